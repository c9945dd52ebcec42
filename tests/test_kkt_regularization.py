"""The KKT regularisation-success path (sqp.py:187-198): a back-substitution
that fails the 1e-10 check, +delta*I on the Hessian diagonal
(delta = reg_scale * max(tr H, 1)), retry, accept.

No trained instance meets it (0 regularisations in 340 reference solves,
SURVEY §7), so the test makes one: the first interior latent of block 0 is
cut out of its decoder (W1[:, 0] = 0 in the subnet and the full map).  Its
Jacobian column is then zero, so H_0 = R_0^T R_0 has a zero row and column
that no constraint row touches: K is exactly singular at every SQP step, the
LU meets a zero pivot, and the regularised K is solvable (the step along the
dead latent is -rho/delta = 0).  Every step takes the retry path, in the
oracle (pinned to the reference below when it is present) and on the device.
"""

import os
import sys

import numpy as np
import pytest

from oracle import ddnm_oracle as O

from .conftest import golden_path
from .test_oracle_golden import rel

REF = "/root/reference/pkg/src"


def _dead_latent_arrays(name="tiny_nm"):
    a = dict(np.load(golden_path(name, "artifacts")))
    for key in ("b0_int_W1", "b0_intf_W1"):
        w = a[key].copy()
        w[:, 0] = 0.0
        a[key] = w
    return a


def _mu():
    return np.array([[1500.0, 9.0], [7200.0, 17.5], [300.0, 22.0]])


def test_oracle_takes_the_regularised_path():
    oi = O.Instance(_dead_latent_arrays())
    for a, lam in _mu():
        r = O.solve(oi, a, lam)
        assert r.regularized >= r.n_iter > 0      # every step took the retry
        assert np.all(np.isfinite(r.x))


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
def test_oracle_regularised_kkt_matches_reference_formula():
    """The oracle's regularised step is the reference's
    assemble_and_solve_kkt on the same K (sqp.py:162-208)."""
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import warnings

    from ddrom.sqp import SqpBlock, SqpProblem, assemble_and_solve_kkt  # noqa: F401
    oi = O.Instance(_dead_latent_arrays())
    a, lam = _mu()[0]
    bbs = oi.boundary(a, lam)
    x0 = O.rbf_query(oi, a, lam)
    lam0 = O.multiplier_least_squares(oi, bbs, x0)
    ev = O.eval_gradients(oi, bbs, x0, lam0)
    s, sl, reg = O.solve_kkt(oi, ev)
    assert reg

    from ddrom.sqp import SqpEval, _BlockEval
    blocks = [_BlockEval(*be, seconds=0.0) for be in ev.blocks]
    rev = SqpEval(rho=ev.rho, con=ev.con, blocks=blocks)
    prob = SqpProblem([SqpBlock(b.n_int, b.n_gam, None, None) for b in oi.blocks], oi.n_c)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        rs, rsl = assemble_and_solve_kkt(prob, rev)
    assert any(issubclass(x.category, RuntimeWarning) for x in w)
    assert rel(s, rs) < 1e-9 and rel(sl, rsl) < 1e-9


@pytest.mark.gpu
def test_device_regularised_path_matches_oracle():
    import paper_2305_15163_b200 as P
    arr = _dead_latent_arrays()
    inst, oi = P.RomInstance(arr), O.Instance(arr)
    mu = _mu()
    res = P.solve_rom_batch(inst, mu)
    for k, (a, lam) in enumerate(mu):
        r = O.solve(oi, a, lam)
        assert r.regularized > 0
        assert res.n_reg[k] == r.regularized, (k, res.n_reg[k], r.regularized)
        assert res.status[k] != P.driver.N.STATUS_KKT_SINGULAR
        assert rel(res.x[k], r.x) < 1e-9 and rel(res.lam[k], r.lam) < 1e-9
        assert res.n_iter[k] == r.n_iter
        # the dead latent never moves from its RBF start (step -rho/delta = 0)
        assert res.x[k][0] == res.x0[k][0]
