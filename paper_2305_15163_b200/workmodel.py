"""Algorithmic work model of the online solve.

Counts the FP64 flops one block evaluation needs (products that are
mu-independent are not counted; exp is counted separately), from the
artifact sizes:

    F = 2|I_h| n + 2 nnz~(n+1) + |I_o|(n+2)              interior subnet + J
      + 2 w_G m + 2 nnz_G (m+1) + N_G (m+2)              interface decoder + J
      + 2 n_C N_G (m+1)                                   WFPC constraint CA g, CA J
      + 20 N_z + 4 nnz_J                                  HR stencil residual + Jacobian
      + 2 (nnz_J^O n + nnz_J^G m)                         chain rule
      + N_z (n+m)(n+m+1) + 2 N_z (n+m) + 2 n_C m          Gram, R^T r, cjac^T lam

and a dense LU KKT solve with one refinement as 2/3 nK^3 + 10 nK^2.
"""

from __future__ import annotations

import numpy as np


def stencil_nnz(arrays: dict, b: int, nx: int, ny: int):
    """(nnz_J, nnz_J interior part) of the dense restricted Jacobian rows of
    block b (partition.py:444-464): columns {p, p+-1, p+-nx} of the row's
    component plus the other component's p."""
    p_ = f"b{b}_"
    rows = arrays[p_ + "res_rows"]
    cols = arrays[p_ + "cols"]
    n_io = arrays[p_ + "io"].size
    n = nx * ny
    local = {int(c): k for k, c in enumerate(cols)}
    tot = inner = 0
    for r in rows:
        r = int(r)
        isv = r >= n
        p = r - n if isv else r
        off = n if isv else 0
        i, j = p % nx, p // nx
        gl = {off + p, (p if isv else n + p)}
        if i > 0:
            gl.add(off + p - 1)
        if i < nx - 1:
            gl.add(off + p + 1)
        if j > 0:
            gl.add(off + p - nx)
        if j < ny - 1:
            gl.add(off + p + nx)
        loc = [local[c] for c in gl]
        tot += len(loc)
        inner += sum(1 for c in loc if c < n_io)
    return tot, inner


def eval_flops(arrays: dict, meta: dict) -> dict:
    n_c = meta["n_c"]
    nx, ny = meta["nx"], meta["ny"]
    per_block, exps = [], 0
    ae = meta["kind"] == "nm"
    for b in range(meta["nblocks"]):
        p = f"b{b}_"
        n, m = meta["n_int"][b], meta["n_gam"][b]
        Io = arrays[p + "io"].size
        Ng = int(arrays[p + "n_interface"])
        Nz = arrays[p + "res_rows"].size
        nnzJ, nnzJ_int = stencil_nnz(arrays, b, nx, ny)
        nnzJ_gam = nnzJ - nnzJ_int
        if ae:
            Ih = arrays[p + "int_b1"].size
            nnz = arrays[p + "int_W2_data"].size
            wg = arrays[p + "gam_b1"].size
            nnzg = arrays[p + "gam_W2_data"].size
            dec = (2 * Ih * n + 2 * nnz * (n + 1) + Io * (n + 2)
                   + 2 * wg * m + 2 * nnzg * (m + 1) + Ng * (m + 2))
            exps += Ih + wg
        else:   # LinearMap: g = Phi x (J = Phi is constant)
            dec = 2 * Io * n + 2 * Ng * m
        F = (dec + 2 * n_c * Ng * (m + 1) + 20 * Nz + 4 * nnzJ
             + 2 * (nnzJ_int * n + nnzJ_gam * m)
             + Nz * (n + m) * (n + m + 1) + 2 * Nz * (n + m) + 2 * n_c * m)
        per_block.append(int(F))
    nK = sum(a + b for a, b in zip(meta["n_int"], meta["n_gam"])) + n_c
    kkt = 2.0 / 3.0 * nK**3 + 10.0 * nK**2
    return {"per_block_eval": per_block, "per_eval": float(np.sum(per_block)),
            "exp_per_eval": int(exps), "kkt": float(kkt), "nK": int(nK)}
