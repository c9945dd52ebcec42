"""Host logic of the batch-wide engine (csrc/ddnm_wide.cu), on the CPU through
ddnm_wide_plan: which instances are eligible, every decoder output lands in
exactly one sweep tile of consecutive outputs, no window union outgrows the
32-unit hidden ring, and the work-item counts follow from the chunk sizes."""

import ctypes as C

import numpy as np
import pytest

import paper_2305_15163_b200 as P
from paper_2305_15163_b200 import _native as N

from .conftest import golden_path


def _plan(name):
    inst = P.RomInstance.load(golden_path(name, "artifacts"))
    art, keep = inst._artifacts_struct()
    info = np.zeros(10, np.int32)
    a = inst.arrays
    nout = sum(int(a[f"b{b}_int_scale"].size + a[f"b{b}_gam_scale"].size) if inst.meta["kind"] == "nm"
               else 0 for b in range(inst.n_blocks))
    tiles = np.full(max(nout, 1), -1, np.int32)
    N.check(N.lib().ddnm_wide_plan(C.byref(art), N.ptr(info, C.c_int32), N.ptr(tiles, C.c_int32)))
    why = N.lib().ddnm_last_error().decode()
    del keep
    return inst, info, tiles[:nout], why


@pytest.mark.parametrize("name", ["tiny_nm", "c0_nm", "c3s_nm", "dd16_nm", "tiny42_nm", "c3_nm", "c4_nm"])
def test_eligible_instances_are_tiled_completely(name):
    inst, info, tiles, _ = _plan(name)
    a = inst.arrays
    assert info[0] == 1
    ntiles, coarse, fine, nrc, ncc, slots, useful, S, maxu = (int(v) for v in info[1:])
    assert np.all(tiles >= 0) and tiles.max() == ntiles - 1
    assert np.all(np.diff(tiles) >= 0) and np.all(np.diff(tiles) <= 1)      # consecutive outputs
    ni, ng = inst.meta["n_int"][0], inst.meta["n_gam"][0]
    T = 4 if max(ni, ng) <= 8 else 2
    assert np.bincount(tiles).max() <= 4
    assert maxu <= 32                                                       # the hidden ring
    nnz = sum(int(a[f"b{b}_int_W2_data"].size + a[f"b{b}_gam_W2_data"].size) for b in range(inst.n_blocks))
    assert useful == nnz and slots >= useful                                 # every entry, once
    assert useful / slots > 0.2                                              # (cnt-specialised loops skip the padding)
    assert S == sum(int(a[f"b{b}_int_scale"].size) * (ni + 1) + int(a[f"b{b}_gam_scale"].size) * (ng + 1)
                    for b in range(inst.n_blocks))
    # parts: coarse ones of ~16 tiles, fine ones of 2; both cover every tile
    assert fine >= coarse >= 2 * inst.n_blocks
    assert -(-ntiles // 2) <= fine <= -(-ntiles // 2) + 2 * inst.n_blocks
    assert nrc == sum(-(-int(a[f"b{b}_res_rows"].size) // 32) for b in range(inst.n_blocks))
    assert ncc == sum(max(1, -(-int(a[f"b{b}_gam_scale"].size) // 64)) for b in range(inst.n_blocks))
    _ = T


@pytest.mark.parametrize("name,reason", [("c0_ls", "linear"), ("tiny_srpc", "SRPC"), ("tiny_nmg", "gappy"),
                                         ("c0_lss", "linear")])
def test_ineligible_instances_say_why(name, reason):
    _, info, _, why = _plan(name)
    assert info[0] == 0 and reason in why


def test_windows_that_are_not_banded_are_refused():
    """A decoder row with a gap in its hidden window (not the reference's banded
    mask) cannot use the ring sweep: not eligible, with the reason."""
    arrays = dict(np.load(golden_path("tiny_nm", "artifacts")))
    idx = arrays["b0_int_W2_indices"].copy()
    ip = arrays["b0_int_W2_indptr"]
    o = int(np.argmax(np.diff(ip) >= 3))
    idx[ip[o] + 1] = idx[ip[o] + 2]                      # a repeated index: no longer k0 + e
    arrays["b0_int_W2_indices"] = idx
    inst = P.RomInstance(arrays)
    art, keep = inst._artifacts_struct()
    info = np.zeros(10, np.int32)
    N.check(N.lib().ddnm_wide_plan(C.byref(art), N.ptr(info, C.c_int32), None))
    assert info[0] == 0 and "contiguous" in N.lib().ddnm_last_error().decode()
    del keep
