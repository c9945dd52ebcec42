"""Parameter and grid types of the Burgers FOM the ROM was built on.

Mirrors ``ddrom.burgers`` (burgers.py:32-106): the domain is
``[-1, 1] x [0, 0.05]`` with central differences (R1/R2);
only the parameter box and the grid geometry are needed online -- the
boundary data itself is evaluated on the device from the closed-form
solution (burgers.py:109-127, 188-210).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

X_MIN, X_MAX = -1.0, 1.0
Y_MIN, Y_MAX = 0.0, 0.05
A_RANGE = (1.0, 1.0e4)
LAM_RANGE = (5.0, 25.0)


@dataclass(frozen=True)
class ParameterPoint:
    """Shock parameters ``(a, lam)`` (burgers.py:44-64)."""

    a: float
    lam: float

    def __post_init__(self):
        if not (np.isfinite(self.a) and np.isfinite(self.lam)):
            raise ValueError("parameters must be finite")
        if not self.in_domain:
            warnings.warn(
                f"parameter ({self.a}, {self.lam}) lies outside the sampled "
                f"box {A_RANGE} x {LAM_RANGE}", stacklevel=3)

    @property
    def in_domain(self) -> bool:
        return (A_RANGE[0] <= self.a <= A_RANGE[1]
                and LAM_RANGE[0] <= self.lam <= LAM_RANGE[1])


@dataclass(frozen=True)
class Grid2D:
    """Uniform interior grid (burgers.py:67-106)."""

    nx: int
    ny: int
    nu: float = 0.1

    def __post_init__(self):
        if self.nx < 2 or self.ny < 2:
            raise ValueError("need nx >= 2 and ny >= 2")
        if not self.nu > 0:
            raise ValueError("viscosity must be positive")

    @property
    def hx(self) -> float:
        return (X_MAX - X_MIN) / (self.nx + 1)

    @property
    def hy(self) -> float:
        return (Y_MAX - Y_MIN) / (self.ny + 1)

    @property
    def nnode(self) -> int:
        return self.nx * self.ny

    @property
    def ndof(self) -> int:
        return 2 * self.nx * self.ny


def seeded_parameters(B: int, seed: int = 0) -> np.ndarray:
    """SURVEY.md §8(d1) parameter draw: a ~ U[1, 1e4], lam ~ U[5, 25]."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(A_RANGE[0], A_RANGE[1], B)
    lam = rng.uniform(LAM_RANGE[0], LAM_RANGE[1], B)
    return np.stack([a, lam], axis=1)


@dataclass(frozen=True, eq=False)
class FomOperators:
    """``ddrom.burgers.FomOperators`` (burgers.py:143-157) for the online
    path: the parameter and grid only.  The device evaluates the boundary
    vectors (burgers.py:188-210) at the sampled rows itself and never
    materialises the global sparse operators, so ``build_problem`` /
    ``init_guess`` read just ``param`` -- a reference ``FomOperators`` is
    accepted wherever this one is."""

    grid: Grid2D
    param: ParameterPoint


def assemble(grid: Grid2D, p: ParameterPoint) -> FomOperators:
    """``ddrom.burgers.assemble`` (burgers.py:174-213) signature; see
    :class:`FomOperators` for what is kept."""
    return FomOperators(grid=grid, param=p)
