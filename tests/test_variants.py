"""SRPC coupling and gappy HR -- oracle pinned to the
reference goldens, CUDA path vs the oracle.

Variants (tools/make_variants.py, tools/make_golden.py):
  *_nmg  NM-ROM, gappy HR (weights = pinv(basis[rows]), hyper.py:153-160)
  *_srpc NM-ROM, SRPC: Sigmoid port nets assembled into the interface maps,
         constraint Ahat x_Gamma (driver.py:374-378), interface decoder
         restricted to the HR rows (driver.py:400-402)
  *_lsg  LS-ROM, gappy HR;  *_lss LS-ROM, SRPC
Per-evaluation pieces are compared tightly.  Whole solves use the
perturbation-calibrated gate of conftest.sensitivity: wherever the oracle is
stable under a 1e-14 perturbation of its start and under another valid KKT
solve, x and lambda must agree to 1e-9 and the trajectory must be identical;
elsewhere the problem itself does not determine x to 1e-9 and the tolerance is
1e3 x that sensitivity (no comparison beyond a sensitivity of 1e-3).
Ill-posed throughout, so their KKT steps are compared through residuals and
their solves through invariants: c0_lsg (gappy bases of 16-45 vectors for 28
latents: H_b = R_b^T R_b is rank deficient, cond(K) ~ 1e18) and c0_srpc
(every trajectory meets a KKT system the reference must regularize: the
trained Sigmoid port nets saturate, leaving latent directions no decoder
output depends on) and c0_lss (SRPC LS-ROM, n = (20, 19), n_C = 40: the
60x60 LS-ROM's H_b already has cond ~ 1e21, SURVEY §7 hard part 2; the
oracle's and the reference's first KKT steps differ by 7% while both solve
K to 1e-10).  c0_lss's 196 x 196 KKT workspace does not fit in shared
memory: it runs the (20, 19) kernels with the KKT workspace in L2 (KG)."""

import numpy as np
import pytest

import paper_2305_15163_b200 as P
from oracle import ddnm_oracle as O

from .conftest import VARIANTS, sensitivity
from .test_oracle_golden import merit_noise, rel

ILL_POSED = {"c0_lsg", "c0_srpc", "c0_lss"}
STEP_TOL = {"tiny_lss": 1e-7, "c0_srpc": 1e-8}   # K amplifies the 1e-13 input round-off
WELL_POSED = [n for n in VARIANTS if n not in ILL_POSED]
MIN_DETERMINED = {"tiny_srpc": 4}


def _kkt_residual(oi, ev, s, sl):
    K = O.kkt_matrix(oi, ev)
    rhs = -ev.optimality
    return float(np.linalg.norm(K @ np.concatenate([s, sl]) - rhs) / np.linalg.norm(rhs))


# -- oracle vs reference ---------------------------------------------------------

@pytest.mark.parametrize("name", VARIANTS)
def test_variant_oracle_eval_and_init(name, oracle_instances, goldens):
    oi, g = oracle_instances[name], goldens[name]
    for k in range(3):
        a, lam = g["mu"][k]
        bbs = oi.boundary(a, lam)
        assert rel(O.rbf_query(oi, a, lam), g["x0"][k]) < 1e-13
        assert rel(O.multiplier_least_squares(oi, bbs, g["x0"][k]), g["lam0"][k]) < 1e-10
        ev = O.eval_gradients(oi, bbs, g["x0"][k], g["lam0"][k])
        assert rel(ev.rho, g[f"d{k}_rho"]) < 1e-12
        assert rel(ev.con, g[f"d{k}_con"]) < 1e-13
        for i, be in enumerate(ev.blocks):
            q = f"d{k}_b{i}_"
            blk = oi.blocks[i]
            xi, xg = oi.split(g["x0"][k])[i]
            if blk.gio.size:
                assert rel(blk.gam_map.decode(xg), g[q + "gam_g"]) < 1e-15
            assert rel(be[0], g[q + "Br"]) < 1e-11
            assert rel(be[1], g[q + "R_int"]) < 1e-13
            assert rel(be[2], g[q + "R_gam"]) < 1e-13
            assert rel(be[3], g[q + "con_val"]) < 1e-13
            assert rel(be[4], g[q + "con_jac"]) < 1e-13
        s, sl, reg = O.solve_kkt(oi, ev)
        assert not reg
        if name in ILL_POSED:
            # both are valid solutions of the (numerically singular) system
            assert _kkt_residual(oi, ev, s, sl) <= 1e-10
            assert _kkt_residual(oi, ev, g[f"d{k}_step"], g[f"d{k}_step_lam"]) <= 1e-8
        else:
            tol = STEP_TOL.get(name, 1e-9)
            assert rel(s, g[f"d{k}_step"]) < tol
            assert rel(sl, g[f"d{k}_step_lam"]) < tol


@pytest.mark.parametrize("name", WELL_POSED)
def test_variant_oracle_solve_matches_reference(name, oracle_instances, goldens):
    oi, g = oracle_instances[name], goldens[name]
    determined = 0
    for k in range(g["mu"].shape[0]):
        sig, r = sensitivity(name, oi, g["mu"][k], g["x0"][k], k)
        if r is None or sig > 1e-3:
            continue              # not determined by the problem at all (diverging)
        tol = max(1e-9, 1e3 * sig)
        determined += tol <= 1e-6
        assert rel(r.x, g["x"][k]) < tol, (k, sig)
        assert rel(r.lam, g["lam"][k]) < tol, (k, sig)
        if sig <= 1e-10 and min(r.margins, default=np.inf) > merit_noise(r.merit_history[0]):
            assert r.n_iter == g["n_iter"][k]
            np.testing.assert_array_equal(r.alpha_history, g["alpha_hist"][k, :r.n_iter])
            assert (r.failure_reason is not None) == bool(g["failure"][k] == 1)
    # most parameters are determined to 1e-6 or better; the SRPC NM-ROMs hit
    # singular KKT systems (saturated Sigmoid port units leave latent
    # directions the decoders ignore) on most trajectories
    assert determined >= MIN_DETERMINED.get(name, 8)


# -- CUDA path vs oracle -------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", VARIANTS)
def test_variant_eval_matches_oracle(name, gpu_instances, oracle_instances, goldens):
    inst, oi, g = gpu_instances[name], oracle_instances[name], goldens[name]
    B = 4
    mu, x, lam = g["mu"][:B], g["x0"][:B], g["lam0"][:B]
    ev = P.eval_gradients_batch(inst, mu, x, lam)
    for k in range(B):
        oev = O.eval_gradients(oi, oi.boundary(*mu[k]), x[k], lam[k])
        assert rel(ev.rho[k], oev.rho) < 1e-11
        assert rel(ev.con[k], oev.con) < 1e-12
        assert abs(ev.merit[k] - oev.merit) <= 1e-11 * oev.merit
        for b, be in enumerate(oev.blocks):
            d = ev.block(k, b)
            blk = oi.blocks[b]
            xi, xg = oi.split(x[k])[b]
            if blk.gio.size or not blk.srpc:
                gg = blk.gam_map.decode(xg)
                assert rel(d["gam_g"], gg if blk.srpc else gg) < 1e-13
            assert rel(d["Br"], be[0]) < 1e-10
            assert rel(d["R_int"], be[1]) < 1e-12
            assert rel(d["R_gam"], be[2]) < 1e-12
            assert rel(d["con_val"], be[3]) < 1e-12
            assert rel(d["con_jac"], be[4]) < 1e-12
        s, sl, reg = O.solve_kkt(oi, oev)
        if name in ILL_POSED:
            nD = oi.n_primal
            assert ev.kkt_status[k] in (0, 1)
            if ev.kkt_status[k] == 0:
                assert _kkt_residual(oi, oev, ev.step[k, :nD], ev.step[k, nD:]) <= 1e-8
        else:
            assert ev.kkt_status[k] == int(reg)
            tol = 10 * STEP_TOL.get(name, 1e-9)
            assert rel(ev.step[k, :oi.n_primal], s) < tol
            assert rel(ev.step[k, oi.n_primal:], sl) < tol


@pytest.mark.gpu
@pytest.mark.parametrize("name", WELL_POSED)
def test_variant_solve_matches_oracle(name, gpu_instances, oracle_instances, goldens):
    inst, oi, g = gpu_instances[name], oracle_instances[name], goldens[name]
    res = P.solve_rom_batch(inst, g["mu"])
    undetermined = 0
    for k in range(g["mu"].shape[0]):
        assert rel(res.x0[k], g["x0"][k]) < 1e-13
        sig, r = sensitivity(name, oi, g["mu"][k], g["x0"][k], k)
        if r is None or 1e3 * sig > 1e-6:
            # the problem does not determine x to 1e-6 at this mu (the oracle
            # moves by more under a 1e-14 start perturbation or another valid
            # KKT solve): no parity claim, counted
            undetermined += 1
            continue
        tol = max(1e-9, 1e3 * sig)          # capped: <= 1e-6
        assert rel(res.x[k], r.x) < tol, (k, sig)
        assert rel(res.lam[k], r.lam) < tol, (k, sig)
        if sig <= 1e-10 and min(r.margins, default=np.inf) > merit_noise(r.merit_history[0]):
            assert res.n_iter[k] == r.n_iter
            np.testing.assert_array_equal(res.alpha_hist[k, :r.n_iter], r.alpha_history)
            assert res.failure_reason(k) == r.failure_reason
    print(f"{name}: {undetermined} of {g['mu'].shape[0]} mu undetermined at 1e-6")
    assert g["mu"].shape[0] - undetermined >= MIN_DETERMINED.get(name, 8)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(ILL_POSED))
def test_ill_posed_variant_solve_invariants(name, gpu_instances, oracle_instances, goldens):
    """No trajectory parity is defined (see module doc); the device solve
    must still satisfy the algorithm's invariants, and its reported merit
    must be the oracle's merit at the device's own final iterate."""
    inst, oi, g = gpu_instances[name], oracle_instances[name], goldens[name]
    cfg = P.SqpConfig()
    res = P.solve_rom_batch(inst, g["mu"])
    for k in range(g["mu"].shape[0]):
        if res.status[k] >= 2:
            continue
        n = res.n_iter[k]
        m = res.merit_hist[k, :n + 1]
        a = res.alpha_hist[k, :n]
        assert np.all(m[1:] <= (1 - cfg.armijo_c1 * a) * m[:-1])
        oev = O.eval_gradients(oi, oi.boundary(*g["mu"][k]), res.x[k], res.lam[k])
        # the merit near a minimiser is a cancellation: compare to the noise
        # floor of the trajectory (1e-13 merit0, SURVEY §7 hard part 1)
        assert abs(oev.merit - res.merit[k]) <= max(1e-9 * oev.merit,
                                                    merit_noise(res.merit_hist[k, 0]))
