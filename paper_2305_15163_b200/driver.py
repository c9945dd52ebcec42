"""Online ROM driver: instances, batched solves and per-block evaluation.

Mirrors the online half of ``ddrom.driver`` (driver.py:93-152, 356-597):

* :class:`RomInstance` -- the artifacts ``build_problem`` consumes
  (driver.py:356-436), loaded from a reference-free ``.npz`` and uploaded
  once per GPU into a ``libddnm`` context;
* :func:`solve_rom_batch` -- ``solve_rom`` (driver.py:554-597,
  ``compute_error=False``) for a whole batch of parameters on the device;
* :func:`solve_rom` / :func:`init_guess` / :func:`build_problem` -- the
  reference's single-parameter entry points, on top of the batched kernel;
* :func:`eval_gradients_batch` -- ``eval_gradients`` (sqp.py:117-146) with
  every intermediate of the HR closure (driver.py:404-432), for parity.
"""

from __future__ import annotations

import ctypes as C
import json
import threading
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .burgers import Grid2D, ParameterPoint
from .errors import ConvergenceError
from .sqp import SqpBlock, SqpConfig, SqpProblem, SqpResult

_FAILURE = {N.STATUS_OK: None, N.STATUS_LINE_SEARCH: "line_search",
            N.STATUS_KKT_SINGULAR: "kkt_singular", N.STATUS_LSTSQ_RANK: "lstsq_rank"}


class RomInstance:
    """Everything the online solve of one DD ROM configuration needs.

    Built from the artifact dictionary written by ``tools/make_golden.py``
    (the reference's ``RomInstance`` after ``attach_hr`` and
    ``fit_initializer``, restricted to what ``build_problem`` reads)."""

    def __init__(self, arrays: dict):
        self.arrays = {k: np.asarray(v) for k, v in arrays.items()}
        self.meta = json.loads(str(self.arrays["meta_json"]))
        m = self.meta
        self.kind = m["kind"]
        self.grid = Grid2D(m["nx"], m["ny"], m["nu"])
        self.n_blocks = m["nblocks"]
        self.latent_layout = [(int(a), int(b)) for a, b in zip(m["n_int"], m["n_gam"])]
        self.n_mult = int(m["n_c"])
        self.n_primal = sum(a + b for a, b in self.latent_layout)
        self.provenance = dict(m.get("provenance", {}))
        self.constraint_mode = m.get("constraint", "wfpc")
        self.srpc = self.constraint_mode == "srpc"
        self.hr_mode = m.get("hr", "collocation")
        self._ctx = {}
        self._lock = threading.Lock()
        self._keep = []

    @classmethod
    def from_ddrom(cls, ref_instance, full_maps: bool = True) -> "RomInstance":
        """From the reference's ``ddrom.driver.RomInstance`` (driver.py:93-152)
        after ``attach_hr``/``fit_initializer`` -- see :mod:`.intake`."""
        from .intake import arrays_from_ddrom
        return cls(arrays_from_ddrom(ref_instance, full_maps=full_maps))

    @classmethod
    def load(cls, path: str) -> "RomInstance":
        """From the ``.npz`` artifacts or a binio instance file pair
        (``.bin`` + ``.txt``, see :mod:`binio`)."""
        if str(path).endswith(".bin"):
            from .binio import load_instance_arrays
            return cls(load_instance_arrays(path))
        with np.load(path, allow_pickle=False) as z:
            return cls(dict(z))

    def save_binio(self, path: str) -> None:
        """Write the artifacts as a binio instance file pair, the input of
        the C entry point ``ddnm_ctx_create_binio``."""
        from .binio import save_instance
        save_instance(self, path)

    def split_latent(self, x):
        out, off = [], 0
        for ni, ng in self.latent_layout:
            out.append((x[off:off + ni], x[off + ni:off + ni + ng]))
            off += ni + ng
        return out

    # -- native context ----------------------------------------------------

    def _artifacts_struct(self):
        a = self.arrays
        m = self.meta
        keep = []

        def arr(x, kind="f"):
            x = N.f64(x) if kind == "f" else N.i64(x)
            keep.append(x)
            return N.ptr(x, C.c_double if kind == "f" else C.c_int64)

        blocks = (N.Block * self.n_blocks)()
        for b in range(self.n_blocks):
            p = f"b{b}_"
            blk = blocks[b]
            blk.n_int, blk.n_gam = self.latent_layout[b]
            io, gio = a[p + "io"], a[p + "gio"]
            self._fill_decoder(blk.interior, p + "int_", arr)
            self._fill_decoder(blk.interface, p + "gam_", arr)
            if self.srpc:
                # the interface decoder is the restriction to gio (driver.py:400-402)
                gio = np.arange(gio.size, dtype=np.int64)
            blk.n_rows = a[p + "res_rows"].size
            blk.res_rows = arr(a[p + "res_rows"], "i")
            blk.n_cols = a[p + "cols"].size
            blk.cols = arr(a[p + "cols"], "i")
            blk.n_io = io.size
            blk.n_gio = gio.size
            blk.gio = arr(gio, "i")
            blk.CA = arr(a[p + "Ahat"] if self.srpc else a[p + "CA"])
            if p + "weights" in a:
                blk.n_basis = a[p + "weights"].shape[0]
                blk.weights = arr(a[p + "weights"])
        art = N.Artifacts()
        art.abi_version = N.ABI_VERSION
        art.map_kind = N.MAP_AUTOENCODER if self.kind == "nm" else N.MAP_LINEAR
        act = m.get("activation", "swish")
        gact = m.get("gam_activation", act)
        art.activation = N.ACT_SIGMOID if act == "sigmoid" else N.ACT_SWISH
        art.gam_activation = N.ACT_SIGMOID if gact == "sigmoid" else N.ACT_SWISH
        art.constraint_mode = N.CON_SRPC if self.srpc else N.CON_WFPC
        art.nx, art.ny, art.nu = m["nx"], m["ny"], m["nu"]
        art.n_blocks = self.n_blocks
        art.n_c = self.n_mult
        art.blocks = blocks
        if "rbf_coeffs" in a:
            if m.get("rbf_kernel", "thin_plate_spline") != "thin_plate_spline":
                raise NotImplementedError("only thin-plate-spline RBF initializers")
            art.rbf.n_centers = a["rbf_y"].shape[0]
            art.rbf.n_mono = a["rbf_powers"].shape[0]
            art.rbf.y = arr(a["rbf_y"])
            art.rbf.coeffs = arr(a["rbf_coeffs"])
            art.rbf.powers = arr(a["rbf_powers"], "i")
            for k in range(2):
                art.rbf.shift[k] = float(a["rbf_shift"][k])
                art.rbf.scale[k] = float(a["rbf_scale"][k])
                art.rbf.lo[k] = float(a["rbf_lo"][k])
                art.rbf.hi[k] = float(a["rbf_hi"][k])
            art.rbf.epsilon = float(m.get("rbf_epsilon", 1.0))
        keep.append(blocks)
        return art, keep

    def _fill_decoder(self, dec, pre, arr):
        a = self.arrays
        if self.kind == "nm":
            dec.n_out = a[pre + "scale"].size
            dec.n_hidden = a[pre + "b1"].size
            dec.W1 = arr(a[pre + "W1"])
            dec.b1 = arr(a[pre + "b1"])
            dec.indptr = arr(a[pre + "W2_indptr"], "i")
            dec.indices = arr(a[pre + "W2_indices"], "i")
            dec.data = arr(a[pre + "W2_data"])
            dec.scale = arr(a[pre + "scale"])
            dec.shift = arr(a[pre + "shift"])
        else:
            Phi = a[pre + "Phi"]
            dec.n_out = Phi.shape[0]
            dec.n_hidden = 0
            dec.W1 = arr(Phi)

    @property
    def has_full_decoders(self) -> bool:
        """Whether the artifacts carry the full interior maps (decode)."""
        return "b0_int_cols" in self.arrays

    @property
    def state_layout(self):
        """[(n_interior_dofs, n_interface_dofs), ...] of RomInstance.decode."""
        a = self.arrays
        return [(int(a[f"b{b}_int_cols"].size), int(a[f"b{b}_gam_cols"].size))
                for b in range(self.n_blocks)]

    def _set_full_decoders(self, h):
        keep = []

        def arr(x, kind="f"):
            x = N.f64(x) if kind == "f" else N.i64(x)
            keep.append(x)
            return N.ptr(x, C.c_double if kind == "f" else C.c_int64)

        decs = (N.Decoder * self.n_blocks)()
        gdecs = (N.Decoder * self.n_blocks)() if self.srpc else None
        for b in range(self.n_blocks):
            self._fill_decoder(decs[b], f"b{b}_intf_", arr)
            if self.srpc:
                self._fill_decoder(gdecs[b], f"b{b}_gamf_", arr)
        N.check(N.lib().ddnm_ctx_set_full_decoders(h, decs, gdecs))

    def decode(self, x, device: int = -1):
        """RomInstance.decode (driver.py:148-152) on the device:
        [(x_int, x_gam), ...] of one latent vector."""
        return decode_batch(self, np.asarray(x, float)[None, :], device=device).blocks(0)

    def restrict_blocks(self, state):
        """driver.py:477-480 (Partition.restrict, partition.py:232-235):
        a global FOM state split into [(x_int, x_gam), ...] per block."""
        state = np.asarray(state, float)
        if state.shape != (self.meta["ndof"],):
            raise ValueError("state has wrong length")
        return [(state[self.arrays[f"b{b}_int_cols"]], state[self.arrays[f"b{b}_gam_cols"]])
                for b in range(self.n_blocks)]

    def assemble_global(self, states):
        """driver.py:483-493: merge per-block states; shared interface entries
        are averaged over the blocks holding them."""
        n = self.meta["ndof"]
        acc, cnt = np.zeros(n), np.zeros(n)
        for b, (xi, xg) in enumerate(states):
            for cols, v in ((self.arrays[f"b{b}_int_cols"], xi),
                            (self.arrays[f"b{b}_gam_cols"], xg)):
                acc[cols] += v
                cnt[cols] += 1
        return acc / np.maximum(cnt, 1)

    def context(self, device: int = -1, slots: int = 0):
        """The libddnm context of this instance on ``device`` (created once)."""
        key = (device, slots)
        with self._lock:
            if key not in self._ctx:
                L = N.lib()
                art, keep = self._artifacts_struct()
                h = C.c_void_p()
                N.check(L.ddnm_ctx_create(device, C.byref(art), slots, C.byref(h)))
                ctx = _Context(h, self)
                if self.has_full_decoders:
                    try:
                        self._set_full_decoders(h)
                    except Exception:
                        ctx.close()
                        raise
                self._ctx[key] = ctx
            return self._ctx[key]

    def close(self):
        with self._lock:
            for c in self._ctx.values():
                c.close()
            self._ctx.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _Context:
    def __init__(self, handle, inst):
        self.h = handle
        self.info = N.Info()
        N.check(N.lib().ddnm_ctx_info(self.h, C.byref(self.info)))

    def close(self):
        if self.h:
            N.lib().ddnm_ctx_destroy(self.h)
            self.h = None

    def profile(self):
        """Per-phase device cycles of the last solve (set DDNM_PROF=1)."""
        buf = (C.c_uint64 * 16)()
        N.check(N.lib().ddnm_last_profile(self.h, buf))
        names = ["fetch", "A_hidden", "B_sweep", "C_stencil", "D_gram", "init", "sqp_state",
                 "kkt"]
        names += ["kkt_factor", "kkt_S", "kkt_solve", "kkt_check", "kkt_setup", "kkt_fallback"]
        return {n: int(buf[i]) for i, n in enumerate(names)}

    def counters(self):
        e, k = C.c_int64(), C.c_int64()
        N.check(N.lib().ddnm_last_counters(self.h, C.byref(e), C.byref(k)))
        return e.value, k.value

    def set_engine(self, engine: str = "auto") -> None:
        """Engine of the batched solve: ``"slots"`` (persistent kernel, one CTA
        slot per mu), ``"wide"`` (one lane per mu, rounds of evaluation and
        SQP-step kernels) or ``"auto"`` (wide when the instance is eligible)."""
        N.check(N.lib().ddnm_ctx_set_engine(self.h, ENGINES[engine]))
        self.engine = engine

    def lanes(self) -> int:
        """Evaluations the wide engine launched in the last solve (with the
        speculative candidates that were not consumed)."""
        n = C.c_int64()
        N.check(N.lib().ddnm_last_lanes(self.h, C.byref(n)))
        return n.value

    def rounds(self):
        """(SQP rounds, kernel launches) of the last batched solve."""
        r, n = C.c_int64(), C.c_int64()
        N.check(N.lib().ddnm_last_rounds(self.h, C.byref(r), C.byref(n)))
        return r.value, n.value


ENGINES = {"auto": 0, "slots": 1, "wide": 2}


def _cfg_struct(cfg: SqpConfig):
    c = N.SqpCfg()
    c.tol, c.max_iter, c.armijo_c1 = cfg.tol, cfg.max_iter, cfg.armijo_c1
    c.backtrack_factor, c.max_halvings = cfg.backtrack_factor, cfg.max_halvings
    c.reg_scale = cfg.reg_scale
    return c


def _mu_array(mus) -> np.ndarray:
    if isinstance(mus, ParameterPoint):
        mus = [mus]
    if isinstance(mus, (list, tuple)) and mus and isinstance(mus[0], ParameterPoint):
        return np.array([[p.a, p.lam] for p in mus], dtype=float)
    mu = np.ascontiguousarray(mus, dtype=float)
    if mu.ndim != 2 or mu.shape[1] != 2:
        raise ValueError("parameters must be an array of shape (B, 2) = (a, lambda)")
    if not np.all(np.isfinite(mu)):
        raise ValueError("parameters must be finite")
    return mu


@dataclass(eq=False)
class BatchResult:
    """Per-parameter outputs of :func:`solve_rom_batch` (row k = mu k)."""

    mu: np.ndarray
    x: np.ndarray
    lam: np.ndarray
    n_iter: np.ndarray
    n_evals: np.ndarray
    status: np.ndarray
    n_reg: np.ndarray
    merit: np.ndarray
    objective: np.ndarray
    merit_hist: np.ndarray
    obj_hist: np.ndarray
    alpha_hist: np.ndarray
    x0: np.ndarray
    lam0: np.ndarray
    seconds: float = 0.0
    tol: float = 1e-4
    counters: tuple = field(default=(0, 0))
    rounds: int = 0        # SQP rounds of the batch-wide engine (0: persistent kernel)
    launches: int = 0      # kernel launches of the solve

    @property
    def converged(self) -> np.ndarray:
        """sqp.py:294-295: merit below tol and no failure."""
        return (self.status == N.STATUS_OK) & (self.merit < self.tol)

    def failure_reason(self, k):
        return _FAILURE[int(self.status[k])]

    def result(self, k: int, cfg: SqpConfig = SqpConfig()) -> SqpResult:
        n = int(self.n_iter[k])
        if int(self.status[k]) == N.STATUS_KKT_SINGULAR:
            raise ConvergenceError("KKT back-substitution residual exceeds 1e-10 after "
                                   "regularization (device solve)")
        if int(self.status[k]) == N.STATUS_LSTSQ_RANK:
            raise ConvergenceError("multiplier least squares is rank deficient: the KKT "
                                   "matrix is singular")
        return SqpResult(
            x=self.x[k].copy(), lam=self.lam[k].copy(), converged=bool(self.converged[k]),
            n_iter=n, merit_history=self.merit_hist[k, :n + 1].tolist(),
            objective_history=self.obj_hist[k, :n + 1].tolist(),
            alpha_history=self.alpha_hist[k, :n].tolist(),
            failure_reason=self.failure_reason(k), n_evals=int(self.n_evals[k]),
            n_regularized=int(self.n_reg[k]))


def _solve_arrays(inst: RomInstance, mu: np.ndarray, cfg: SqpConfig, x0=None, lam0=None,
                  device: int = -1, slots: int = 0, engine: str = "auto") -> BatchResult:
    if engine not in ENGINES:
        raise ValueError(f"engine must be one of {sorted(ENGINES)}")
    ctx = inst.context(device, slots)
    prev = getattr(ctx, "engine", "auto")          # a choice made on the context stays
    ctx.set_engine(engine if engine != "auto" else prev)
    B = mu.shape[0]
    nD, nC, K = inst.n_primal, inst.n_mult, cfg.max_iter
    out = dict(
        x=np.empty((B, nD)), lam=np.empty((B, nC)), n_iter=np.zeros(B, np.int32),
        n_evals=np.zeros(B, np.int32), status=np.zeros(B, np.int32),
        n_reg=np.zeros(B, np.int32), merit=np.empty(B), objective=np.empty(B),
        merit_hist=np.empty((B, K + 1)), obj_hist=np.empty((B, K + 1)),
        alpha_hist=np.empty((B, K)), x0=np.empty((B, nD)), lam0=np.empty((B, nC)))
    so = N.SolveOut()
    for k, v in out.items():
        setattr(so, k, N.ptr(v, C.c_int32 if v.dtype == np.int32 else C.c_double))
    if x0 is not None:
        x0 = N.f64(x0).reshape(B, nD)
    if lam0 is not None:
        lam0 = N.f64(lam0).reshape(B, nC)
    t0 = time.perf_counter()
    try:
        N.check(N.lib().ddnm_solve_batch(ctx.h, B, N.ptr(mu), N.ptr(x0), N.ptr(lam0),
                                         C.byref(_cfg_struct(cfg)), C.byref(so)))
    finally:
        ctx.set_engine(prev)
    dt = time.perf_counter() - t0
    rounds, launches = ctx.rounds()
    return BatchResult(mu=mu, seconds=dt, tol=cfg.tol, counters=ctx.counters(), rounds=rounds,
                       launches=launches, **out)


def solve_rom_batch(instance: RomInstance, mus, cfg: SqpConfig = SqpConfig(), *,
                    x0=None, lam0=None, device: int = -1, slots: int = 0,
                    engine: str = "auto") -> BatchResult:
    """``solve_rom`` (driver.py:554-597, compute_error=False) for every mu.

    ``mus``: (B, 2) array of (a, lambda) or a list of ParameterPoint.
    ``x0``/``lam0``: optional (B, n_D) / (B, n_C) starting points; when absent
    the device evaluates the RBF initializer (driver.py:82-90) and the
    least-squares multipliers (driver.py:461-471), as ``init_guess`` does.
    ``engine``: ``"auto"`` (the batch-wide kernels when the instance is
    eligible, else the persistent kernel), ``"slots"`` or ``"wide"``."""
    mu = _mu_array(mus)
    span_lo = instance.arrays.get("rbf_lo")
    if x0 is None and span_lo is not None:
        lo, hi = instance.arrays["rbf_lo"], instance.arrays["rbf_hi"]
        span = np.where(hi > lo, hi - lo, 1.0)
        qn = (mu - lo) / span
        if np.any(qn < -0.1) or np.any(qn > 1.1):
            warnings.warn("initializing far outside the training box", RuntimeWarning,
                          stacklevel=2)
    return _solve_arrays(instance, mu, cfg, x0, lam0, device, slots, engine)


@dataclass(eq=False)
class DecodeBatch:
    """Decoded states of a batch (row k = mu k), flattened per mu as
    [blk0 interior | blk0 interface | blk1 interior | ...]."""

    states: np.ndarray
    layout: list
    error: np.ndarray = None

    def blocks(self, k: int):
        """RomInstance.decode's list of (x_int, x_gam) for mu k."""
        out, off = [], 0
        for ni, ng in self.layout:
            out.append((self.states[k, off:off + ni], self.states[k, off + ni:off + ni + ng]))
            off += ni + ng
        return out


def decode_batch(instance: RomInstance, x, *, fom_states=None, device: int = -1,
                 keep_states: bool = True) -> DecodeBatch:
    """RomInstance.decode (driver.py:148-152) of every latent row of ``x`` on
    the device; with ``fom_states`` ((B, ndof) global FOM states) also
    relative_error (driver.py:496-507) of each row against
    restrict_blocks(fom_states[k]) (driver.py:477-480)."""
    if not instance.has_full_decoders:
        raise ValueError("the artifacts carry no full interior maps (regenerate them with "
                         "tools/make_golden.py)")
    x = N.f64(x)
    if x.ndim != 2 or x.shape[1] != instance.n_primal:
        raise ValueError("latents must have shape (B, n_primal)")
    B = x.shape[0]
    layout = instance.state_layout
    L = sum(a + b for a, b in layout)
    ctx = instance.context(device)
    states = np.empty((B, L)) if keep_states else None
    fom = err = None
    if fom_states is not None:
        fs = np.asarray(fom_states, float)
        if fs.shape != (B, instance.meta["ndof"]):
            raise ValueError("fom_states must have shape (B, ndof)")
        cols = np.concatenate([np.concatenate([instance.arrays[f"b{b}_int_cols"],
                                               instance.arrays[f"b{b}_gam_cols"]])
                               for b in range(instance.n_blocks)])
        fom = N.f64(fs[:, cols])
        err = np.empty(B)
    N.check(N.lib().ddnm_decode_batch(ctx.h, B, N.ptr(x), N.ptr(fom), N.ptr(states),
                                      N.ptr(err)))
    if err is not None and np.isnan(err).any():
        raise ValueError("zero-norm reference block")
    return DecodeBatch(states=states, layout=layout, error=err)


@dataclass(eq=False)
class RomSolution:
    """driver.py:513-519."""

    x_latent: np.ndarray
    lam: np.ndarray
    states: list = field(repr=False, default=None)
    sqp: SqpResult = field(repr=False, default=None)
    error: float = np.nan


@dataclass(eq=False)
class BenchmarkRecord:
    """driver.py:522-551 (same fields, CSV header and row)."""

    label: str
    config: dict
    a: float
    lam: float
    error: float = np.nan
    fom_seconds: float = np.nan
    rom_seconds: float = np.nan
    parallel_seconds: float = np.nan
    per_iter_seconds: float = np.nan
    speedup: float = np.nan
    n_iter: int = 0
    converged: bool = False
    final_merit: float = np.nan
    status: str = "ok"

    HEADER = ["label", "rom", "constraint", "hr", "n_int", "n_gam", "a",
              "lambda", "error", "fom_seconds", "rom_seconds",
              "parallel_seconds", "per_iter_seconds", "speedup", "n_iter",
              "converged", "final_merit", "status"]

    def row(self):
        c = self.config
        return [self.label, c.get("rom", ""), c.get("constraint", ""),
                c.get("hr", ""), c.get("n_int", ""), c.get("n_gam", ""),
                self.a, self.lam, self.error, self.fom_seconds,
                self.rom_seconds, self.parallel_seconds,
                self.per_iter_seconds, self.speedup, self.n_iter,
                int(self.converged), self.final_merit, self.status]


def _param_of(ops_or_p) -> ParameterPoint:
    """The parameter of a ``FomOperators`` (ours or the reference's:
    burgers.py:143-157 carries ``param``) or a ``ParameterPoint``."""
    if isinstance(ops_or_p, ParameterPoint):
        return ops_or_p
    p = getattr(ops_or_p, "param", None)
    if p is None or not hasattr(p, "a") or not hasattr(p, "lam"):
        raise ValueError("expected FomOperators (assemble(grid, p)) or a ParameterPoint")
    return p if isinstance(p, ParameterPoint) else ParameterPoint(float(p.a), float(p.lam))


def solve_rom(instance: RomInstance, p: ParameterPoint, cfg: SqpConfig = SqpConfig(), *,
              x0=None, lam0=None, fom_state=None, fom_seconds: float = np.nan,
              compute_error: bool = True, label: str = ""):
    """Solve the ROM at ``p`` (driver.py:554-597) on the GPU; returns
    ``(RomSolution, BenchmarkRecord)`` like the reference.

    ``compute_error`` (default True, as the reference): without ``fom_state``
    the full-order solution is computed first on the host (``fom.py``, the
    reference's own ``solve_monolithic`` path, driver.py:566-569; not part of
    the ROM solve and not in ``rom_seconds``), then ``error`` =
    ``relative_error`` of the device decode (driver.py:589-592).  The record's
    ``parallel_seconds`` is the device time of the solve (every block of an
    evaluation runs concurrently on the GPU, the execution model the
    reference emulates with its max-over-blocks charge, driver.py:580)."""
    part_fom = None
    if compute_error and fom_state is None:
        from .fom import solve_monolithic
        t0 = time.perf_counter()
        part_fom = solve_monolithic(instance.grid, p)
        fom_seconds = time.perf_counter() - t0
        fom_state = part_fom
    if compute_error and not instance.has_full_decoders:
        raise ValueError("compute_error needs the full decoders (artifacts with *_intf_* maps)")
    mu = np.array([[p.a, p.lam]], dtype=float)
    res = solve_rom_batch(instance, mu, cfg,
                          x0=None if x0 is None else np.asarray(x0, float)[None, :],
                          lam0=None if lam0 is None else np.asarray(lam0, float)[None, :])
    r = res.result(0, cfg)
    states, error = None, np.nan
    if instance.has_full_decoders:
        dec = decode_batch(instance, r.x[None, :],
                           fom_states=(None if not compute_error or fom_state is None
                                       else np.asarray(fom_state)[None]))
        states = dec.blocks(0)
        if dec.error is not None:
            error = float(dec.error[0])
    parallel = float(res.seconds)
    rec = BenchmarkRecord(
        label=label or instance.provenance.get("rom", "rom"), config=dict(instance.provenance),
        a=p.a, lam=p.lam, error=error, fom_seconds=fom_seconds, rom_seconds=parallel,
        parallel_seconds=parallel, per_iter_seconds=parallel / max(r.n_iter, 1),
        speedup=fom_seconds / parallel if parallel > 0 else np.nan,
        n_iter=r.n_iter, converged=r.converged, final_merit=r.final_merit,
        status="ok" if r.failure_reason is None else r.failure_reason)
    return RomSolution(x_latent=r.x, lam=r.lam, states=states, sqp=r, error=error), rec


def init_guess(instance: RomInstance, p: ParameterPoint, *, ops=None, prob=None):
    """RBF latents plus least-squares multipliers (driver.py:442-458),
    evaluated on the device.  ``ops`` / ``prob`` are accepted as in the
    reference (they only let it reuse assembled operators); the device reads
    the parameter alone."""
    if ops is not None and _param_of(ops) != p:
        raise ValueError("ops were assembled at a different parameter")
    if prob is not None and getattr(prob, "param", p) != p:
        raise ValueError("problem was built at a different parameter")
    mu = np.array([[p.a, p.lam]], dtype=float)
    res = solve_rom_batch(instance, mu, SqpConfig(max_iter=1, tol=1e300))
    return res.x0[0].copy(), res.lam0[0].copy()


@dataclass(eq=False)
class EvalBatch:
    rho: np.ndarray
    con: np.ndarray
    merit: np.ndarray
    objective: np.ndarray
    Br: np.ndarray
    R: np.ndarray
    cval: np.ndarray
    cjac: np.ndarray
    int_g: np.ndarray
    int_J: np.ndarray
    gam_g: np.ndarray
    gam_J: np.ndarray
    bvals: np.ndarray
    step: np.ndarray
    kkt_status: np.ndarray
    layout: dict = field(default_factory=dict)

    def block(self, k: int, b: int) -> dict:
        """Per-block views for mu k, block b, in the reference's shapes."""
        L = self.layout[b]
        ni, ng = L["n_int"], L["n_gam"]
        w = ni + ng
        r0, r1 = L["row"]
        o0, o1 = L["out"]
        R = self.R[k, L["R"][0]:L["R"][1]].reshape(o1 - o0, w)
        return {
            "Br": self.Br[k, o0:o1], "R_int": R[:, :ni], "R_gam": R[:, ni:],
            "con_val": self.cval[k, b], "con_jac": self.cjac[k, L["cjac"][0]:L["cjac"][1]]
            .reshape(-1, ng),
            "int_g": self.int_g[k, L["iout"][0]:L["iout"][1]],
            "int_J": self.int_J[k, L["intJ"][0]:L["intJ"][1]].reshape(-1, ni),
            "gam_g": self.gam_g[k, L["gout"][0]:L["gout"][1]],
            "gam_J": self.gam_J[k, L["gamJ"][0]:L["gamJ"][1]].reshape(-1, ng),
            "bvals": self.bvals[k, r0:r1],
        }


def eval_gradients_batch(instance: RomInstance, mus, x, lam, *, reg_scale: float = 1e-12,
                         step: bool = True, device: int = -1) -> EvalBatch:
    """``eval_gradients`` (sqp.py:117-146) at (x[k], lam[k]) for every mu,
    with all HR-closure intermediates, and optionally the KKT step
    (sqp.py:162-208) at that point."""
    mu = _mu_array(mus)
    B = mu.shape[0]
    ctx = instance.context(device)
    inf = ctx.info
    nD, nC = inf.n_primal, inf.n_mult
    x = N.f64(x).reshape(B, nD)
    lam = N.f64(lam).reshape(B, nC)
    o = dict(rho=np.empty((B, nD)), con=np.empty((B, nC)), merit=np.empty(B),
             objective=np.empty(B), Br=np.empty((B, inf.total_out_rows)),
             R=np.empty((B, inf.total_out_R)), cval=np.empty((B, inf.n_blocks, nC)),
             cjac=np.empty((B, inf.total_cjac)), int_g=np.empty((B, inf.total_int_out)),
             int_J=np.empty((B, inf.total_int_J)), gam_g=np.empty((B, inf.total_gam_out)),
             gam_J=np.empty((B, inf.total_gam_J)), bvals=np.empty((B, inf.total_rows, 3)),
             step=np.empty((B, nD + nC)) if step else None,
             kkt_status=np.zeros(B, np.int32) if step else None)
    eo = N.EvalOut()
    for k, v in o.items():
        if v is not None:
            setattr(eo, k, N.ptr(v, C.c_int32 if v.dtype == np.int32 else C.c_double))
    N.check(N.lib().ddnm_eval_batch(ctx.h, B, N.ptr(mu), N.ptr(x), N.ptr(lam), reg_scale,
                                    C.byref(eo)))
    layout, offs = {}, dict(row=0, out=0, R=0, cjac=0, iout=0, intJ=0, gout=0, gamJ=0)
    a = instance.arrays
    for b, (ni, ng) in enumerate(instance.latent_layout):
        p = f"b{b}_"
        nrows = a[p + "res_rows"].size
        nout = a[p + "weights"].shape[0] if p + "weights" in a else nrows
        nio = a[p + "io"].size
        ngo = a[p + "gio"].size if instance.srpc else int(a[p + "n_interface"])
        sizes = dict(row=nrows, out=nout, R=nout * (ni + ng), cjac=nC * ng, iout=nio,
                     intJ=nio * ni, gout=ngo, gamJ=ngo * ng)
        layout[b] = {"n_int": ni, "n_gam": ng}
        for key, sz in sizes.items():
            layout[b][key] = (offs[key], offs[key] + sz)
            offs[key] += sz
    return EvalBatch(layout=layout, **o)


def build_problem(instance: RomInstance, ops) -> SqpProblem:
    """``build_problem(instance, ops)`` (driver.py:356-436): blocks whose
    residual/constraint closures evaluate on the GPU (one eval per call), so
    the reference's own ``sqp.iterate`` can drive them.  ``ops`` is
    ``assemble(grid, p)`` (ours or the reference's); a ``ParameterPoint`` is
    accepted too."""
    p = _param_of(ops)
    mu = np.array([[p.a, p.lam]], dtype=float)
    offs = np.cumsum([0] + [a + b for a, b in instance.latent_layout])
    nD, nC = instance.n_primal, instance.n_mult
    blocks = []
    for b, (ni, ng) in enumerate(instance.latent_layout):
        def _eval(xi, xg, b=b, ni=ni, ng=ng):
            x = np.zeros(nD)
            x[offs[b]:offs[b] + ni] = xi
            x[offs[b] + ni:offs[b] + ni + ng] = xg
            ev = eval_gradients_batch(instance, mu, x[None], np.zeros((1, nC)), step=False)
            return ev.block(0, b)

        def residual(xi, xg, _e=_eval):
            d = _e(np.asarray(xi, float), np.asarray(xg, float))
            return d["Br"].copy(), d["R_int"].copy(), d["R_gam"].copy()

        def constraint(xg, _e=_eval, ni=ni):
            d = _e(np.zeros(ni), np.asarray(xg, float))
            return d["con_val"].copy(), d["con_jac"].copy()

        blocks.append(SqpBlock(ni, ng, residual, constraint))
    return SqpProblem(blocks, nC, instance=instance, param=p)
