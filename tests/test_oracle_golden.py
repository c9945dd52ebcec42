"""Pin the CPU oracle (oracle/ddnm_oracle.py) to the reference's own outputs.

tests/golden/*_golden.npz were produced by tools/make_golden.py running the
reference package (ddrom) on the same artifacts; nothing here imports it."""

import numpy as np
import pytest

from oracle import ddnm_oracle as O

from .conftest import BIG, N_BIG, N_ORACLE, NAMES, n_detail


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)) if b.size else 0.0


@pytest.mark.parametrize("name", NAMES)
def test_init_guess_matches_reference(name, oracle_instances, goldens):
    inst, g = oracle_instances[name], goldens[name]
    for k in range(4):
        a, lam = g["mu"][k]
        bbs = inst.boundary(a, lam)
        assert rel(O.rbf_query(inst, a, lam), g["x0"][k]) < 1e-13       # driver.py:82-90
        lam0 = O.multiplier_least_squares(inst, bbs, g["x0"][k])          # driver.py:461-471
        assert rel(lam0, g["lam0"][k]) < 1e-12


@pytest.mark.parametrize("name", NAMES)
def test_eval_pieces_match_reference(name, oracle_instances, goldens):
    inst, g = oracle_instances[name], goldens[name]
    for k in range(n_detail(g)):
        a, lam = g["mu"][k]
        bbs = inst.boundary(a, lam)
        ev = O.eval_gradients(inst, bbs, g["x0"][k], g["lam0"][k])
        assert rel(ev.rho, g[f"d{k}_rho"]) < 1e-12
        assert rel(ev.con, g[f"d{k}_con"]) < 1e-13
        assert abs(ev.merit - g[f"d{k}_merit"]) <= 1e-12 * g[f"d{k}_merit"]
        for i, be in enumerate(ev.blocks):
            q = f"d{k}_b{i}_"
            # boundary vectors are bitwise (same closed form, same numpy ops)
            np.testing.assert_array_equal(bbs[i][0], g[q + "bx"])
            np.testing.assert_array_equal(bbs[i][1], g[q + "by"])
            np.testing.assert_array_equal(bbs[i][2], g[q + "bc"])
            blk = inst.blocks[i]
            xi, xg = inst.split(g["x0"][k])[i]
            if blk.n_io:
                assert rel(blk.int_map.decode(xi), g[q + "int_g"]) < 1e-15
                assert rel(blk.int_map.jacobian(xi), g[q + "int_J"]) < 1e-15
            assert rel(blk.gam_map.decode(xg), g[q + "gam_g"]) < 1e-15
            assert rel(blk.gam_map.jacobian(xg), g[q + "gam_J"]) < 1e-15
            assert rel(be[0], g[q + "Br"]) < 1e-11
            assert rel(be[1], g[q + "R_int"]) < 1e-13
            assert rel(be[2], g[q + "R_gam"]) < 1e-13
            assert rel(be[3], g[q + "con_val"]) < 1e-13
            assert rel(be[4], g[q + "con_jac"]) < 1e-13


@pytest.mark.parametrize("name", NAMES)
def test_kkt_step_matches_reference(name, oracle_instances, goldens):
    inst, g = oracle_instances[name], goldens[name]
    for k in range(n_detail(g)):
        a, lam = g["mu"][k]
        ev = O.eval_gradients(inst, inst.boundary(a, lam), g["x0"][k], g["lam0"][k])
        s, sl, reg = O.solve_kkt(inst, ev)
        assert not reg
        # cond(K) ~ 1e20-1e24: steps agree to far below the 1e-9 gate
        assert rel(s, g[f"d{k}_step"]) < 1e-9
        assert rel(sl, g[f"d{k}_step_lam"]) < 1e-9


# oracle-vs-reference iteration-count agreement where it is not every mu
# (decided by round-off at the merit floor, SURVEY §7 hard part 1)
ITER_AGREEMENT = {"c0_ls": 7, "c3s_nm": 15}


def merit_noise(merit0):
    """Absolute round-off floor of the merit: ~1e-13 * merit0 (SURVEY §0
    finding 2: ~1e-3 absolute at 60x60 where merit0 ~ 1e10)."""
    return 1e-13 * merit0


@pytest.mark.parametrize("name", NAMES)
def test_solve_matches_reference(name, oracle_instances, goldens):
    """x, lam to 1e-9 relative always; n_iter, alpha history and failure flag
    identical whenever no tol/Armijo decision on the path was within the merit
    noise floor (SURVEY §7 hard part 1: the margin-aware gate)."""
    inst, g = oracle_instances[name], goldens[name]
    B = N_ORACLE.get(name, g["mu"].shape[0])
    robust = same_iters = 0
    for k in range(B):
        a, lam = g["mu"][k]
        r = O.solve(inst, a, lam)
        assert rel(r.x, g["x"][k]) < 1e-9
        assert rel(r.lam, g["lam"][k]) < 1e-9
        if min(r.margins) > merit_noise(r.merit_history[0]):
            robust += 1
            assert r.n_iter == g["n_iter"][k]
            np.testing.assert_array_equal(r.alpha_history, g["alpha_hist"][k, :r.n_iter])
            np.testing.assert_allclose(r.merit_history, g["merit_hist"][k, :r.n_iter + 1],
                                       rtol=1e-9, atol=merit_noise(r.merit_history[0]))
            assert (r.failure_reason is not None) == bool(g["failure"][k] == 1)
        same_iters += int(r.n_iter == g["n_iter"][k])
    # c0_ls: every trajectory touches the noise floor (cond(H_i) ~ 1e21,
    # SURVEY §7 hard part 2) -- only the 1e-9 state gate applies there
    assert robust >= (0 if name == "c0_ls" else 1)
    # iteration counts equal to the reference's on every mu, except where a
    # tol/Armijo decision sits at the merit round-off floor (measured: c0_ls
    # 7/16 -- config 1 claims no iteration-count parity -- and c3s_nm 15/16)
    assert same_iters >= ITER_AGREEMENT.get(name, B), (name, same_iters)
