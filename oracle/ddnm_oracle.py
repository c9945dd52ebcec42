"""CPU oracle: a numpy restatement of the reference's online DD NM-ROM-HR solve.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` leg may import this module,
and only as the checker or the timed CPU baseline -- never as the product
path.  The product (``paper_2305_15163_b200``) runs the hand-written CUDA
kernels and fails loudly when they are missing.

Parity pin: every function here is checked in ``tests/test_oracle_golden.py``
against ``tests/golden/*_golden.npz``, which ``tools/make_golden.py`` produced
by running the reference package itself (``/root/reference/pkg/src/ddrom``)
on the same artifacts.  The third-party numerics the reference calls are
numpy 2.3.5 / scipy 1.18.1 (``pyproject.toml:9-13``): ``lu_factor/lu_solve``
(LAPACK getrf/getrs), ``np.linalg.lstsq`` (gelsd) and scipy's
``RBFInterpolator`` evaluation; this restatement calls the same routines.

Reference map (file:line under ``/root/reference/pkg/src/ddrom``):

* ``exact_solution``           burgers.py:109-127
* ``boundary_values``          burgers.py:188-210 (ghost-point vectors)
* ``act`` / ``act_deriv``      autoencoder.py:31-45
* ``SparseDecoder``            hyper.py:163-197, autoencoder.py:134-163
* ``LinearDecoder``            pod.py:67-97
* ``Stencil``                  partition.py:350-464 (RestrictedResidual)
* ``Block.residual``           driver.py:404-432 (collocation HR closure)
* ``Block.constraint``         driver.py:371-373 (WFPC)
* ``eval_gradients``           sqp.py:117-146
* ``solve_kkt``                sqp.py:149-208
* ``iterate``                  sqp.py:230-299
* ``rbf_query``                driver.py:82-90 + scipy _rbfinterp evaluation
* ``multiplier_least_squares`` driver.py:461-471
* ``solve``                    driver.py:554-597 (compute_error=False path)
"""

from __future__ import annotations

import json
import warnings
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse
from scipy.special import expit

X_MIN, X_MAX = -1.0, 1.0          # burgers.py:32-33
Y_MIN, Y_MAX = 0.0, 0.05


class OracleConvergenceError(RuntimeError):
    """Mirror of ``errors.ConvergenceError`` (errors.py:8-13)."""


# -- PDE pieces -----------------------------------------------------------

def exact_solution(a, lam, x, y, nu=0.1):
    """burgers.py:109-127."""
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    ep = np.exp(lam * (x - 1.0))
    em = np.exp(-lam * (x - 1.0))
    cy = np.cos(lam * y)
    sy = np.sin(lam * y)
    psi = a * (1.0 + x) + (ep + em) * cy
    if np.any(np.abs(psi) < 1e-300):
        raise ValueError("psi vanishes at an evaluation point")
    u = -2.0 * nu * (a + lam * (ep - em) * cy) / psi
    v = 2.0 * nu * lam * (ep + em) * sy / psi
    return u, v


def grid_steps(nx, ny):
    return (X_MAX - X_MIN) / (nx + 1), (Y_MAX - Y_MIN) / (ny + 1)


def boundary_values(nx, ny, nu, a, lam):
    """The six mu-dependent vectors of ``assemble`` (burgers.py:188-210)."""
    hx, hy = grid_steps(nx, ny)
    n = nx * ny
    xs = X_MIN + hx * np.arange(1, nx + 1)
    ys = hy * np.arange(1, ny + 1)
    uL, vL = exact_solution(a, lam, X_MIN, ys, nu)
    uR, vR = exact_solution(a, lam, X_MAX, ys, nu)
    uB, vB = exact_solution(a, lam, xs, Y_MIN, nu)
    uT, vT = exact_solution(a, lam, xs, Y_MAX, nu)
    left = np.arange(ny) * nx
    right = left + (nx - 1)
    bottom = np.arange(nx)
    top = (ny - 1) * nx + np.arange(nx)

    def edge(gL, gR, gB, gT):
        exl = np.zeros(n); exl[left] = gL
        exr = np.zeros(n); exr[right] = gR
        eyb = np.zeros(n); eyb[bottom] = gB
        eyt = np.zeros(n); eyt[top] = gT
        bx = (-1.0 / (2.0 * hx)) * (exl - exr)
        by = (-1.0 / (2.0 * hy)) * (eyb - eyt)
        c = (nu / hx**2) * (exl + exr) + (nu / hy**2) * (eyb + eyt)
        return bx, by, c

    bux, buy, cu = edge(uL, uR, uB, uT)
    bvx, bvy, cv = edge(vL, vR, vB, vT)
    return bux, buy, cu, bvx, bvy, cv


# -- decoders ---------------------------------------------------------------

def act(tag, z):
    """autoencoder.py:31-36."""
    if tag == "swish":
        return z * expit(z)
    if tag == "sigmoid":
        return expit(z)
    raise ValueError(tag)


def act_deriv(tag, z):
    """autoencoder.py:39-45."""
    s = expit(z)
    if tag == "swish":
        return s * (1.0 + z * (1.0 - s))
    if tag == "sigmoid":
        return s * (1.0 - s)
    raise ValueError(tag)


@dataclass(eq=False)
class SparseDecoder:
    """Shallow sparse decoder / subnet (hyper.py:163-197).

    Hidden layer accumulated latent column by latent column (hyper.py:184-188),
    output layer a CSR row sweep in storage order (hyper.py:190-197)."""

    W1: np.ndarray
    b1: np.ndarray
    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray
    scale: np.ndarray
    shift: np.ndarray
    activation: str = "swish"

    @property
    def latent_dim(self):
        return self.W1.shape[1]

    @property
    def out_dim(self):
        return self.scale.size

    def _hidden(self, xhat):
        z = self.b1.copy()
        for d in range(self.W1.shape[1]):
            z += self.W1[:, d] * xhat[d]
        return z

    def _csr(self, v):
        # CSR row sweep in storage order (scipy csr matvec, as the reference)
        W2 = scipy.sparse.csr_matrix((self.data, self.indices, self.indptr),
                                     shape=(self.out_dim, self.W1.shape[0]))
        return W2 @ v.reshape(self.W1.shape[0], -1)

    def decode(self, xhat):
        a = act(self.activation, self._hidden(np.asarray(xhat, dtype=float)))
        return self._csr(a)[:, 0] * self.scale + self.shift

    def jacobian(self, xhat):
        zp = act_deriv(self.activation,
                       self._hidden(np.asarray(xhat, dtype=float)))
        return self._csr(zp[:, None] * self.W1) * self.scale[:, None]


@dataclass(eq=False)
class LinearDecoder:
    """``LinearMap`` (pod.py:67-97): g = Phi x, J = Phi."""

    Phi: np.ndarray

    @property
    def latent_dim(self):
        return self.Phi.shape[1]

    def decode(self, xhat):
        return self.Phi @ xhat

    def jacobian(self, xhat=None):
        return self.Phi


# -- restricted stencil -------------------------------------------------------

class Stencil:
    """Selected Burgers residual rows from a local column vector
    (``RestrictedResidual``, partition.py:350-464), dense Jacobian."""

    def __init__(self, nx, ny, nu, rows, cols):
        hx, hy = grid_steps(nx, ny)
        n = nx * ny
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        self.rows, self.cols, self.n = rows, cols, n
        lookup = np.full(2 * n, -1, dtype=np.int64)
        lookup[cols] = np.arange(cols.size)
        cx = -1.0 / (2.0 * hx)
        cyy = -1.0 / (2.0 * hy)
        dx = nu / hx**2
        dy = nu / hy**2
        self.terms = []     # per row: (gu, gv, Bx[(c,w)], By[(c,w)], Cd[(c,w)])
        self.node = np.empty(rows.size, np.int64)
        self.isu = rows < n
        for r in rows:
            p = int(r if r < n else r - n)
            off = 0 if r < n else n
            i, j = p % nx, p // nx
            bx, by, cd = [], [], []
            if i > 0:
                bx.append((p - 1, cx * -1.0))
            if i < nx - 1:
                bx.append((p + 1, cx * 1.0))
            if j > 0:
                by.append((p - nx, cyy * -1.0))
            if j < ny - 1:
                by.append((p + nx, cyy * 1.0))
            if j > 0:
                cd.append((p - nx, dy * 1.0))
            if i > 0:
                cd.append((p - 1, dx * 1.0))
            cd.append((p, dx * -2.0 + dy * -2.0))
            if i < nx - 1:
                cd.append((p + 1, dx * 1.0))
            if j < ny - 1:
                cd.append((p + nx, dy * 1.0))

            def loc(lst):
                out = []
                for c, w in lst:
                    lc = lookup[c + off]
                    if lc < 0:
                        raise ValueError("restricted rows reference columns "
                                         "outside the provided column set")
                    out.append((int(lc), w))
                return out
            gu, gv = lookup[p], lookup[p + n]
            if gu < 0 or gv < 0:
                raise ValueError("diagonal coupling column missing")
            self.terms.append((int(gu), int(gv), loc(bx), loc(by), loc(cd)))
        self.node = np.where(self.isu, rows, rows - n)

    def boundary(self, bvec):
        """Per-row (bx, by, c) sliced from the six ``assemble`` vectors
        (partition.py:404-415)."""
        bux, buy, cu, bvx, bvy, cv = bvec
        nd = self.node
        return (np.where(self.isu, bux[nd], bvx[nd]),
                np.where(self.isu, buy[nd], bvy[nd]),
                np.where(self.isu, cu[nd], cv[nd]))

    def residual(self, x, bb):
        bx, by, c = bb
        out = np.empty(self.rows.size)
        for k, (gu, gv, tx, ty, tc) in enumerate(self.terms):
            sx = sum(w * x[q] for q, w in tx)
            sy = sum(w * x[q] for q, w in ty)
            sc = sum(w * x[q] for q, w in tc)
            out[k] = x[gu] * (sx - bx[k]) + x[gv] * (sy - by[k]) + sc + c[k]
        return out

    def jacobian(self, x, bb):
        bx, by, _ = bb
        J = np.zeros((self.rows.size, self.cols.size))
        for k, (gu, gv, tx, ty, tc) in enumerate(self.terms):
            sx = sum(w * x[q] for q, w in tx)
            sy = sum(w * x[q] for q, w in ty)
            J[k, gu] += sx - bx[k]
            J[k, gv] += sy - by[k]
            for q, w in tx:
                J[k, q] += x[gu] * w
            for q, w in ty:
                J[k, q] += x[gv] * w
            for q, w in tc:
                J[k, q] += w
        return J


# -- instance -------------------------------------------------------------------

@dataclass(eq=False)
class Block:
    n_int: int
    n_gam: int
    int_map: object
    gam_map: object
    gio: np.ndarray
    n_io: int
    CA: np.ndarray            # WFPC: C @ A_i [n_c x N_Gamma]; SRPC: Ahat_i [n_c x n_gam]
    stencil: Stencil
    srpc: bool = False        # interface map = subnet on the gio outputs (driver.py:400-402)
    weights: np.ndarray = None  # gappy HR: pinv of the sampled residual basis

    def residual(self, xi, xg, bb):
        """HR closure (driver.py:404-432): collocation, or gappy weighting
        ``weights @`` of the sampled residual and Jacobian (hyper.py:107-118)."""
        if self.n_io:
            v_int = self.int_map.decode(xi)
            J_int_rows = np.asarray(self.int_map.jacobian(xi))
        else:
            v_int = np.zeros(0)
            J_int_rows = None
        if self.gio.size and self.srpc:
            v_gam = self.gam_map.decode(xg)
            J_gam_rows = np.asarray(self.gam_map.jacobian(xg))
        elif self.gio.size:
            g = self.gam_map.decode(xg)
            J = np.asarray(self.gam_map.jacobian(xg))
            v_gam, J_gam_rows = g[self.gio], J[self.gio]
        else:
            v_gam, J_gam_rows = np.zeros(0), np.zeros((0, self.n_gam))
        v = np.concatenate([v_int, v_gam])
        r = self.stencil.residual(v, bb)
        Jd = self.stencil.jacobian(v, bb)
        if J_int_rows is not None:
            R_int = Jd[:, :self.n_io] @ J_int_rows
        else:
            R_int = np.zeros((Jd.shape[0], self.n_int))
        R_gam = Jd[:, self.n_io:] @ J_gam_rows
        if self.weights is not None:
            return self.weights @ r, self.weights @ R_int, self.weights @ R_gam
        return r, R_int, R_gam

    def constraint(self, xg):
        """WFPC (driver.py:371-373) or SRPC (driver.py:374-378) constraint."""
        if self.srpc:
            return self.CA @ xg, self.CA.copy()
        g = self.gam_map.decode(xg)
        J = np.asarray(self.gam_map.jacobian(xg))
        return self.CA @ g, self.CA @ J


class Instance:
    """Everything the online solve consumes, from an artifact ``.npz``."""

    def __init__(self, path_or_dict):
        d = (dict(np.load(path_or_dict, allow_pickle=False))
             if isinstance(path_or_dict, str) else path_or_dict)
        self.raw = d
        m = json.loads(str(d["meta_json"]))
        self.meta = m
        self.kind = m["kind"]
        self.nx, self.ny, self.nu = m["nx"], m["ny"], m["nu"]
        self.n_c = m["n_c"]
        self.blocks = []
        for b in range(m["nblocks"]):
            p = f"b{b}_"
            ni, ng = m["n_int"][b], m["n_gam"][b]
            io, gio = d[p + "io"], d[p + "gio"]
            if self.kind == "nm":
                im = SparseDecoder(d[p + "int_W1"], d[p + "int_b1"],
                                   d[p + "int_W2_indptr"], d[p + "int_W2_indices"],
                                   d[p + "int_W2_data"], d[p + "int_scale"],
                                   d[p + "int_shift"], m["activation"])
                gm = SparseDecoder(d[p + "gam_W1"], d[p + "gam_b1"],
                                   d[p + "gam_W2_indptr"], d[p + "gam_W2_indices"],
                                   d[p + "gam_W2_data"], d[p + "gam_scale"],
                                   d[p + "gam_shift"],
                                   m.get("gam_activation", m["activation"]))
            else:
                im = LinearDecoder(d[p + "int_Phi"])
                gm = LinearDecoder(d[p + "gam_Phi"])
            st = Stencil(self.nx, self.ny, self.nu, d[p + "res_rows"],
                         d[p + "cols"])
            srpc = m.get("constraint", "wfpc") == "srpc"
            self.blocks.append(Block(ni, ng, im, gm, gio, int(io.size),
                                     d[p + "Ahat"] if srpc else d[p + "CA"], st, srpc,
                                     d.get(p + "weights")))
        self.offsets = np.cumsum([0] + [b.n_int + b.n_gam
                                        for b in self.blocks])[:-1]
        self.n_primal = int(sum(b.n_int + b.n_gam for b in self.blocks))
        self.rbf = {k[4:]: d[k] for k in d if k.startswith("rbf_")}
        # full interior maps + dof columns for decode / restrict (optional keys)
        self.full_interior = []
        self.cols = []
        for b in range(m["nblocks"]):
            p = f"b{b}_"
            if p + "int_cols" not in d:
                self.full_interior = None
                break
            full = []
            for pre, act in (("intf_", m["activation"]),
                             ("gamf_", m.get("gam_activation", m["activation"]))):
                if pre == "gamf_" and p + pre + "scale" not in d and p + pre + "Phi" not in d:
                    full.append(self.blocks[b].gam_map)     # WFPC: gam_ is the full map
                elif self.kind == "nm":
                    full.append(SparseDecoder(
                        d[p + pre + "W1"], d[p + pre + "b1"], d[p + pre + "W2_indptr"],
                        d[p + pre + "W2_indices"], d[p + pre + "W2_data"],
                        d[p + pre + "scale"], d[p + pre + "shift"], act))
                else:
                    full.append(LinearDecoder(d[p + pre + "Phi"]))
            self.full_interior.append(tuple(full))
            self.cols.append((d[p + "int_cols"], d[p + "gam_cols"]))

    def decode(self, x):
        """RomInstance.decode (driver.py:148-152): [(x_int, x_gam), ...]."""
        if self.full_interior is None:
            raise ValueError("artifacts carry no full interior maps")
        return [(fi.decode(xi), fg.decode(xg))
                for (fi, fg), (xi, xg) in zip(self.full_interior, self.split(x))]

    def restrict_blocks(self, state):
        """driver.py:477-480 / Partition.restrict (partition.py:232-235)."""
        return [(state[ci], state[cg]) for ci, cg in self.cols]

    def split(self, x):
        return [(x[o:o + b.n_int], x[o + b.n_int:o + b.n_int + b.n_gam])
                for o, b in zip(self.offsets, self.blocks)]

    def boundary(self, a, lam):
        bvec = boundary_values(self.nx, self.ny, self.nu, a, lam)
        return [b.stencil.boundary(bvec) for b in self.blocks]


def relative_error(fom_blocks, rom_blocks):
    """driver.py:496-507: root mean over blocks of the squared blockwise
    relative error."""
    if len(fom_blocks) != len(rom_blocks):
        raise ValueError("block counts differ")
    total = 0.0
    for (fi, fg), (ri, rg) in zip(fom_blocks, rom_blocks):
        denom = float(fi @ fi + fg @ fg)
        if denom == 0.0:
            raise ValueError("zero-norm reference block")
        total += float((fi - ri) @ (fi - ri) + (fg - rg) @ (fg - rg)) / denom
    return float(np.sqrt(total / len(fom_blocks)))


# -- SQP --------------------------------------------------------------------------

@dataclass
class SqpConfig:
    """sqp.py:68-81."""
    tol: float = 1e-4
    max_iter: int = 15
    armijo_c1: float = 1e-4
    backtrack_factor: float = 0.5
    max_halvings: int = 25
    reg_scale: float = 1e-12


@dataclass(eq=False)
class Eval:
    rho: np.ndarray
    con: np.ndarray
    blocks: list = field(default_factory=list)   # (Br, R_int, R_gam, cval, cjac)

    @property
    def optimality(self):
        return np.concatenate([self.rho, self.con])

    @property
    def merit(self):
        return float(np.linalg.norm(self.optimality))

    @property
    def objective(self):
        return 0.5 * sum(float(b[0] @ b[0]) for b in self.blocks)


def eval_gradients(inst: Instance, bbs, x, lam) -> Eval:
    """sqp.py:117-146."""
    rho = np.zeros(inst.n_primal)
    con = np.zeros(inst.n_c)
    evals = []
    for blk, bb, off, (xi, xg) in zip(inst.blocks, bbs, inst.offsets,
                                      inst.split(x)):
        Br, R_int, R_gam = blk.residual(xi, xg, bb)
        cval, cjac = blk.constraint(xg)
        cjac = np.atleast_2d(cjac)
        rho[off:off + blk.n_int] = R_int.T @ Br
        rho[off + blk.n_int:off + blk.n_int + blk.n_gam] = (
            R_gam.T @ Br + cjac.T @ lam)
        con += cval
        evals.append((Br, R_int, R_gam, cval, cjac))
    return Eval(rho=rho, con=con, blocks=evals)


def kkt_matrix(inst: Instance, ev: Eval):
    """sqp.py:149-159."""
    n, m = inst.n_primal, inst.n_c
    K = np.zeros((n + m, n + m))
    for off, blk, be in zip(inst.offsets, inst.blocks, ev.blocks):
        R = np.hstack([be[1], be[2]])
        w = blk.n_int + blk.n_gam
        K[off:off + w, off:off + w] = R.T @ R
        gs = off + blk.n_int
        K[n:, gs:gs + blk.n_gam] = be[4]
        K[gs:gs + blk.n_gam, n:] = be[4].T
    return K


def solve_kkt(inst: Instance, ev: Eval, reg_scale=1e-12, equilibrate=False, noise=None):
    """sqp.py:162-208; returns (s, s_lam, regularized).

    Test instruments (not the reference's algorithm), used by the tests to
    measure how much a problem's trajectory depends on round-off in the
    linear solve: ``equilibrate`` factors the row-equilibrated system D K
    (another valid FP64 solve of the same equations); ``noise`` (a numpy
    Generator) perturbs the Hessian diagonal by one unit round-off of each
    row's largest entry, the backward error any stable LU is allowed."""
    n = inst.n_primal
    K = kkt_matrix(inst, ev)
    if noise is not None:
        rmax = np.max(np.abs(K[:n, :n]), axis=1)
        K[np.arange(n), np.arange(n)] += 1.1e-16 * rmax * noise.standard_normal(n)
    rhs = -ev.optimality
    rhs_norm = max(np.linalg.norm(rhs), 1e-300)

    def attempt(mat):
        if equilibrate:
            dr = 1.0 / np.maximum(np.max(np.abs(mat), axis=1), 1e-300)
            lu, piv = scipy.linalg.lu_factor(mat * dr[:, None])
            pivot = float(np.abs(np.diag(lu)).min())
            sol = scipy.linalg.lu_solve((lu, piv), rhs * dr)
            if not np.all(np.isfinite(sol)):
                return sol, np.inf, pivot
            sol += scipy.linalg.lu_solve((lu, piv), (rhs - mat @ sol) * dr)
            if not np.all(np.isfinite(sol)):
                return sol, np.inf, pivot
            return sol, np.linalg.norm(rhs - mat @ sol) / rhs_norm, pivot
        lu, piv = scipy.linalg.lu_factor(mat)
        pivot = float(np.abs(np.diag(lu)).min())
        sol = scipy.linalg.lu_solve((lu, piv), rhs)
        if not np.all(np.isfinite(sol)):
            return sol, np.inf, pivot
        sol += scipy.linalg.lu_solve((lu, piv), rhs - mat @ sol)
        if not np.all(np.isfinite(sol)):
            return sol, np.inf, pivot
        return sol, np.linalg.norm(rhs - mat @ sol) / rhs_norm, pivot

    reg = False
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            sol, res, pivot = attempt(K)
        ok = res <= 1e-10
    except scipy.linalg.LinAlgError:
        sol, res, pivot, ok = None, np.inf, 0.0, False
    if not ok:
        reg = True
        delta = reg_scale * max(np.trace(K[:n, :n]), 1.0)
        K[np.arange(n), np.arange(n)] += delta
        try:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                sol, res, pivot = attempt(K)
        except scipy.linalg.LinAlgError as exc:
            raise OracleConvergenceError("KKT matrix is singular") from exc
        if res > 1e-10:
            raise OracleConvergenceError(
                f"KKT back-substitution residual {res:.3e} exceeds 1e-10")
    return sol[:n], sol[n:], reg


@dataclass(eq=False)
class Result:
    x: np.ndarray
    lam: np.ndarray
    converged: bool
    n_iter: int
    merit_history: list
    objective_history: list
    alpha_history: list
    failure_reason: str | None = None
    n_evals: int = 0
    regularized: int = 0
    # absolute decision gaps |lhs - rhs| of every tol / Armijo test taken
    margins: list = field(default_factory=list)


def iterate(inst: Instance, bbs, x0, lam0, cfg=SqpConfig(), equilibrate=False,
            noise=None) -> Result:
    """sqp.py:230-299 (plus an eval counter and decision margins)."""
    x = np.array(x0, dtype=float)
    lam = np.array(lam0, dtype=float)
    ev = eval_gradients(inst, bbs, x, lam)
    n_evals = 1
    merits, objectives, alphas = [ev.merit], [ev.objective], []
    best = (ev.merit, x.copy(), lam.copy())
    failure = None
    margins = []
    n_iter = 0
    regs = 0
    while True:
        margins.append(abs(merits[-1] - cfg.tol))
        if not (merits[-1] >= cfg.tol and n_iter < cfg.max_iter):
            break
        s, s_lam, reg = solve_kkt(inst, ev, cfg.reg_scale, equilibrate, noise)
        regs += int(reg)
        alpha = 1.0
        accepted = None
        for _ in range(cfg.max_halvings + 1):
            trial = eval_gradients(inst, bbs, x + alpha * s, lam + alpha * s_lam)
            n_evals += 1
            rhs = (1.0 - cfg.armijo_c1 * alpha) * merits[-1]
            margins.append(abs(trial.merit - rhs))
            if trial.merit <= rhs:
                accepted = trial
                break
            alpha *= cfg.backtrack_factor
        if accepted is None:
            failure = "line_search"
            break
        x += alpha * s
        lam += alpha * s_lam
        ev = accepted
        n_iter += 1
        merits.append(ev.merit)
        objectives.append(ev.objective)
        alphas.append(alpha)
        if ev.merit < best[0]:
            best = (ev.merit, x.copy(), lam.copy())
    if failure is not None:
        _, x, lam = best
    return Result(x=x, lam=lam,
                  converged=bool(merits[-1] < cfg.tol) and failure is None,
                  n_iter=n_iter, merit_history=merits,
                  objective_history=objectives, alpha_history=alphas,
                  failure_reason=failure, n_evals=n_evals, regularized=regs,
                  margins=margins)


# -- initialization -------------------------------------------------------------

def rbf_query(inst: Instance, a, lam):
    """driver.py:82-90 + scipy RBFInterpolator evaluation
    (thin-plate spline, degree-1 polynomial tail)."""
    r = inst.rbf
    q = np.array([a, lam], dtype=float)
    span = np.where(r["hi"] > r["lo"], r["hi"] - r["lo"], 1.0)
    qn = (q - r["lo"]) / span
    eps = float(inst.meta["rbf_epsilon"])
    if inst.meta["rbf_kernel"] != "thin_plate_spline":
        raise NotImplementedError(inst.meta["rbf_kernel"])
    dist = np.linalg.norm(qn[None, :] * eps - r["y"] * eps, axis=-1)
    with np.errstate(divide="ignore", invalid="ignore"):
        ker = np.where(dist == 0, 0, dist**2 * np.log(dist))
    xhat = (qn - r["shift"]) / r["scale"]
    poly = np.prod(xhat[None, :] ** r["powers"], axis=-1)
    vec = np.concatenate([ker, poly])
    return vec @ r["coeffs"]


def multiplier_least_squares(inst: Instance, bbs, x0):
    """driver.py:461-471."""
    ev = eval_gradients(inst, bbs, x0, np.zeros(inst.n_c))
    rows, rhs = [], []
    for off, blk, be in zip(inst.offsets, inst.blocks, ev.blocks):
        gs = off + blk.n_int
        rows.append(be[4].T)
        rhs.append(-ev.rho[gs:gs + blk.n_gam])
    lam, *_ = np.linalg.lstsq(np.vstack(rows), np.concatenate(rhs), rcond=None)
    return lam


def solve(inst: Instance, a, lam_mu, cfg=SqpConfig(), x0=None, lam0=None,
          equilibrate=False, noise=None):
    """driver.py:554-597 without the FOM error (compute_error=False)."""
    bbs = inst.boundary(a, lam_mu)
    if x0 is None:
        x0 = rbf_query(inst, a, lam_mu)
        lam_ls = multiplier_least_squares(inst, bbs, x0)
        lam0 = lam_ls if lam0 is None else lam0
    elif lam0 is None:
        lam0 = multiplier_least_squares(inst, bbs, np.asarray(x0, float))
    return iterate(inst, bbs, x0, lam0, cfg, equilibrate, noise)
