"""Full-order reference solution for the error metric of ``solve_rom``.

``ddrom.driver.solve_rom`` (driver.py:566-569) defaults to
``compute_error=True``: without a given ``fom_state`` it solves the
full-order model (``burgers.solve_monolithic``, burgers.py:281-337: damped
Newton with a sparse LU per step) and reports ``relative_error`` against it.
That FOM solve is not part of the ROM's online path ("FOM
Newton ... OUT OF SCOPE"); it runs on the host here exactly as in the
reference -- the ROM solve itself never does.  Same discretisation
(burgers.py:174-237: central differences on [-1, 1] x [0, 0.05], ghost
values from the closed-form solution), same Newton loop and stopping rule.
"""

from __future__ import annotations

import numpy as np

from .burgers import X_MAX, X_MIN, Y_MAX, Y_MIN, Grid2D, ParameterPoint
from .errors import ConvergenceError


def exact_solution(p: ParameterPoint, x, y, nu: float = 0.1):
    """Cole-Hopf closed form (burgers.py:109-127)."""
    a, lam = p.a, p.lam
    ep, em = np.exp(lam * (x - 1.0)), np.exp(-lam * (x - 1.0))
    cy, sy = np.cos(lam * y), np.sin(lam * y)
    psi = a * (1.0 + x) + (ep + em) * cy
    u = -2.0 * nu * (a + lam * (ep - em) * cy) / psi
    v = 2.0 * nu * lam * (ep + em) * sy / psi
    return u, v


def _operators(grid: Grid2D, p: ParameterPoint):
    import scipy.sparse as sp
    nx, ny, nu, hx, hy, n = grid.nx, grid.ny, grid.nu, grid.hx, grid.hy, grid.nnode

    def d1(m):
        e = np.ones(m - 1)
        return sp.diags([-e, e], [-1, 1], format="csr")

    def d2(m):
        e = np.ones(m)
        return sp.diags([e[:-1], -2.0 * e, e[:-1]], [-1, 0, 1], format="csr")
    Bx = (-1.0 / (2.0 * hx)) * sp.kron(sp.identity(ny), d1(nx), format="csr")
    By = (-1.0 / (2.0 * hy)) * sp.kron(d1(ny), sp.identity(nx), format="csr")
    Cd = ((nu / hx**2) * sp.kron(sp.identity(ny), d2(nx))
          + (nu / hy**2) * sp.kron(d2(ny), sp.identity(nx))).tocsr()
    xs = X_MIN + hx * np.arange(1, nx + 1)
    ys = Y_MIN + hy * np.arange(1, ny + 1)
    uL, vL = exact_solution(p, X_MIN, ys, nu)
    uR, vR = exact_solution(p, X_MAX, ys, nu)
    uB, vB = exact_solution(p, xs, Y_MIN, nu)
    uT, vT = exact_solution(p, xs, Y_MAX, nu)
    left = np.arange(ny) * nx
    right = left + (nx - 1)
    bottom = np.arange(nx)
    top = (ny - 1) * nx + np.arange(nx)

    def edge(gL, gR, gB, gT):
        exl = np.zeros(n); exl[left] = gL
        exr = np.zeros(n); exr[right] = gR
        eyb = np.zeros(n); eyb[bottom] = gB
        eyt = np.zeros(n); eyt[top] = gT
        return ((-1.0 / (2.0 * hx)) * (exl - exr), (-1.0 / (2.0 * hy)) * (eyb - eyt),
                (nu / hx**2) * (exl + exr) + (nu / hy**2) * (eyb + eyt))
    return Bx, By, Cd, edge(uL, uR, uB, uT), edge(vL, vR, vB, vT)


def solve_monolithic(grid: Grid2D, p: ParameterPoint, tol: float = 1e-8, max_iter: int = 25):
    """Damped Newton on the FOM (burgers.py:281-337); returns the state."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    Bx, By, Cd, (bux, buy, cu), (bvx, bvy, cv) = _operators(grid, p)
    n = grid.nnode

    def residual(s):
        u, v = s[:n], s[n:]
        ru = u * (Bx @ u - bux) + v * (By @ u - buy) + Cd @ u + cu
        rv = u * (Bx @ v - bvx) + v * (By @ v - bvy) + Cd @ v + cv
        return np.concatenate([ru, rv])

    def jacobian(s):
        u, v = s[:n], s[n:]
        D = sp.diags
        Juu = D(Bx @ u - bux) + D(u) @ Bx + D(v) @ By + Cd
        Juv = D(By @ u - buy)
        Jvu = D(Bx @ v - bvx)
        Jvv = D(u) @ Bx + D(By @ v - bvy) + D(v) @ By + Cd
        return sp.bmat([[Juu, Juv], [Jvu, Jvv]], format="csc")

    s = np.zeros(grid.ndof)
    r = residual(s)
    rn = float(np.linalg.norm(r))
    for _ in range(max_iter):
        if rn <= tol:
            return s
        d = spla.splu(jacobian(s)).solve(-r)
        alpha = 1.0
        for _h in range(21):
            sn = s + alpha * d
            rnew = residual(sn)
            rnn = float(np.linalg.norm(rnew))
            if rnn < rn:
                break
            alpha *= 0.5
        else:
            raise ConvergenceError(f"Newton stagnated at |r| = {rn:.3e}")
        s, r, rn = sn, rnew, rnn
    if rn <= tol:
        return s
    raise ConvergenceError(f"no convergence in {max_iter} iterations (|r| = {rn:.3e})")
