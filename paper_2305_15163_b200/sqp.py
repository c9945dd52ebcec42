"""SQP configuration, results and the problem/block duck types.

Mirrors ``ddrom.sqp`` (sqp.py:28-299).  The solver loop itself runs on the
device (``csrc/ddnm_solve.cuh``: the Armijo line search, best-iterate
fallback, KKT LU with one refinement and the +delta*I regularisation retry);
:func:`iterate` here drives it for one problem, and :class:`SqpBlock` /
:class:`SqpProblem` expose the same per-block evaluator surface as the
reference so its own ``iterate`` can drive GPU block evaluations for
parity debugging.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True, eq=False)
class SqpBlock:
    """One subdomain's evaluators (sqp.py:28-41)."""

    n_int: int
    n_gam: int
    residual: object
    constraint: object


class SqpProblem:
    """Block-separable problem (sqp.py:44-65); ``instance``/``param`` link it
    to the device context that evaluates it."""

    def __init__(self, blocks, n_mult: int, *, instance=None, param=None):
        if not blocks:
            raise ValueError("need at least one block")
        if n_mult < 0:
            raise ValueError("multiplier dimension must be nonnegative")
        self.blocks = list(blocks)
        self.n_mult = n_mult
        self.offsets = []
        pos = 0
        for b in self.blocks:
            self.offsets.append(pos)
            pos += b.n_int + b.n_gam
        self.n_primal = pos
        self.instance = instance
        self.param = param

    def split(self, x):
        out = []
        for off, b in zip(self.offsets, self.blocks):
            out.append((x[off:off + b.n_int],
                        x[off + b.n_int:off + b.n_int + b.n_gam]))
        return out


@dataclass(frozen=True)
class SqpConfig:
    """sqp.py:68-81 (same defaults and validation)."""

    tol: float = 1e-4
    max_iter: int = 15
    armijo_c1: float = 1e-4
    backtrack_factor: float = 0.5
    max_halvings: int = 25
    reg_scale: float = 1e-12
    record_iterates: bool = True

    def __post_init__(self):
        if (self.tol <= 0 or self.max_iter < 1 or self.armijo_c1 <= 0
                or not 0 < self.backtrack_factor < 1 or self.max_halvings < 0):
            raise ValueError("invalid solver configuration")


@dataclass(eq=False)
class SqpResult:
    """sqp.py:211-227.  ``iterates``/``steps``/``timings`` are not recorded by
    the device loop (the loop never leaves the GPU); ``n_evals`` and
    ``n_regularized`` are extra device counters."""

    x: np.ndarray
    lam: np.ndarray
    converged: bool
    n_iter: int
    merit_history: list
    objective_history: list
    alpha_history: list
    failure_reason: str | None = None
    iterates: list = field(default_factory=list, repr=False)
    steps: list = field(default_factory=list, repr=False)
    timings: dict = field(default_factory=dict, repr=False)
    n_evals: int = 0
    n_regularized: int = 0

    @property
    def final_merit(self) -> float:
        return self.merit_history[-1]


def iterate(prob: SqpProblem, x0, lam0=None, cfg: SqpConfig = SqpConfig()) -> SqpResult:
    """Run the device SQP loop for one problem from ``(x0, lam0)``
    (sqp.py:230-299).  ``prob`` must come from :func:`driver.build_problem`."""
    from .driver import _solve_arrays
    if prob.instance is None:
        raise ValueError("problem was not built by paper_2305_15163_b200.build_problem")
    x = np.array(x0, dtype=float)
    if x.shape != (prob.n_primal,):
        raise ValueError("initial point has wrong length")
    lam = (np.zeros(prob.n_mult) if lam0 is None else np.array(lam0, dtype=float))
    if lam.shape != (prob.n_mult,):
        raise ValueError("initial multiplier has wrong length")
    if not (np.all(np.isfinite(x)) and np.all(np.isfinite(lam))):
        raise ValueError("initial point must be finite")
    p = prob.param
    res = _solve_arrays(prob.instance, np.array([[p.a, p.lam]]), cfg, x[None, :],
                        lam[None, :])
    return res.result(0, cfg)
