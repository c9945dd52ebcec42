"""Evaluation units (blocks split into chunks of sampled rows and chunks of
interface outputs, the device path of configs 3/4) against whole-block
evaluation, the oracle and the reference goldens.

Forcing the split on the small instances (DDNM_UNIT_ROWS) runs the same
code the 480^2 / 960^2 instances need, against goldens that exist for every
intermediate: every decoder value, Jacobian row, residual row and R row is
bitwise the whole block's (a unit's subnet restricts the block's subnet once
more, extract_subnet hyper.py:200-222, so each kept output is computed from
the same entries in the same order); Gram blocks and constraint values are
sums taken chunk by chunk, equal to rounding."""

import numpy as np
import pytest

import paper_2305_15163_b200 as P

from .conftest import golden_path
from .test_oracle_golden import rel

pytestmark = pytest.mark.gpu

SPLIT = ["tiny_nm", "c0_nm", "c3s_nm", "dd16_nm"]


def _whole_instance(name, monkeypatch):
    """Every block evaluated whole (DDNM_NO_UNITS), whatever its size."""
    monkeypatch.setenv("DDNM_NO_UNITS", "1")
    inst = P.RomInstance.load(golden_path(name, "artifacts"))
    ctx = inst.context()
    monkeypatch.delenv("DDNM_NO_UNITS")
    assert ctx.info.eval_units == 0
    return inst


def _split_instance(name, monkeypatch, rows="24", gam="64"):
    monkeypatch.setenv("DDNM_UNIT_ROWS", rows)
    monkeypatch.setenv("DDNM_UNIT_GAM", gam)
    inst = P.RomInstance.load(golden_path(name, "artifacts"))
    ctx = inst.context()
    monkeypatch.delenv("DDNM_UNIT_ROWS")
    monkeypatch.delenv("DDNM_UNIT_GAM")
    assert ctx.info.eval_units > inst.n_blocks
    return inst


@pytest.mark.parametrize("name", SPLIT)
def test_units_eval_match_whole_blocks(name, gpu_instances, goldens, monkeypatch):
    whole, g = _whole_instance(name, monkeypatch), goldens[name]
    split = _split_instance(name, monkeypatch)
    B = 5
    mu, x, lam = g["mu"][:B], g["x0"][:B], g["lam0"][:B]
    ew = P.eval_gradients_batch(whole, mu, x, lam)
    es = P.eval_gradients_batch(split, mu, x, lam)
    for k in range(B):
        for b in range(whole.n_blocks):
            dw, ds = ew.block(k, b), es.block(k, b)
            for key in ("int_g", "int_J", "gam_g", "gam_J", "Br", "R_int", "R_gam", "bvals"):
                np.testing.assert_array_equal(ds[key], dw[key], err_msg=f"{key} mu {k} block {b}")
            assert rel(ds["con_val"], dw["con_val"]) < 1e-13
            assert rel(ds["con_jac"], dw["con_jac"]) < 1e-13
        assert rel(es.rho[k], ew.rho[k]) < 1e-12
        assert rel(es.con[k], ew.con[k]) < 1e-12          # sum over blocks: cancellation
        assert abs(es.merit[k] - ew.merit[k]) <= 1e-12 * ew.merit[k]
        assert rel(es.step[k], ew.step[k]) < 1e-8
        assert rel(es.rho[k], g[f"d{k}_rho"]) < 1e-11 if f"d{k}_rho" in g else True


@pytest.mark.parametrize("name", SPLIT)
def test_units_solve_match_reference(name, gpu_instances, goldens, monkeypatch):
    whole, g = _whole_instance(name, monkeypatch), goldens[name]
    split = _split_instance(name, monkeypatch)
    rw = P.solve_rom_batch(whole, g["mu"], engine="slots")
    rs = P.solve_rom_batch(split, g["mu"], engine="slots")
    for k in range(g["mu"].shape[0]):
        if g["failure"][k] == 2:
            continue
        assert rel(rs.x[k], g["x"][k]) < 1e-9, k
        assert rel(rs.lam[k], g["lam"][k]) < 1e-9, k
        assert rel(rs.x[k], rw.x[k]) < 1e-9, k
    # the merit floor decides iteration counts only at knife-edge mu; the
    # split and whole evaluations agree on (almost) all of them
    assert np.mean(rs.n_iter == rw.n_iter) >= 0.75


def test_units_batch_composition_invariance(monkeypatch):
    """Split evaluation stays deterministic: a mu alone or in a batch is bitwise equal."""
    split = _split_instance("c0_nm", monkeypatch)
    mu = P.seeded_parameters(40, seed=9)
    full = P.solve_rom_batch(split, mu, engine="slots")
    for k in (0, 13, 39):
        one = P.solve_rom_batch(split, mu[k:k + 1], engine="slots")
        np.testing.assert_array_equal(one.x[0], full.x[k])
        np.testing.assert_array_equal(one.lam[0], full.lam[k])


@pytest.mark.parametrize("name", ["c0_nm", "c3_nm", "tiny42_nm"])
def test_tensor_core_hidden_layer_matches_oracle(name, goldens, oracle_instances, monkeypatch):
    """The hidden pre-activation on the FP64 tensor cores (hidden_range,
    DDNM_HIDDEN_DMMA=1; opt-in): decoder values and
    Jacobians to 1e-13 against the oracle, solves to 1e-9 against the
    reference goldens."""
    from oracle import ddnm_oracle as O
    monkeypatch.setenv("DDNM_HIDDEN_DMMA", "1")
    inst = P.RomInstance.load(golden_path(name, "artifacts"))
    inst.context()
    monkeypatch.delenv("DDNM_HIDDEN_DMMA")
    g, oi = goldens[name], oracle_instances[name]
    ev = P.eval_gradients_batch(inst, g["mu"][:3], g["x0"][:3], g["lam0"][:3])
    for k in range(3):
        for b, blk in enumerate(oi.blocks):
            d = ev.block(k, b)
            xi, xg = oi.split(g["x0"][k])[b]
            assert rel(d["int_g"], blk.int_map.decode(xi)) < 1e-13
            assert rel(d["int_J"], blk.int_map.jacobian(xi)) < 1e-13
            assert rel(d["gam_g"], blk.gam_map.decode(xg)) < 1e-13
            assert rel(d["gam_J"], blk.gam_map.jacobian(xg)) < 1e-13
        assert rel(ev.rho[k], O.eval_gradients(oi, oi.boundary(*g["mu"][k]), g["x0"][k],
                                               g["lam0"][k]).rho) < 1e-11
    res = P.solve_rom_batch(inst, g["mu"], engine="slots")     # the slot kernels' hidden layer
    for k in range(g["mu"].shape[0]):
        assert rel(res.x[k], g["x"][k]) < 1e-9 and rel(res.lam[k], g["lam"][k]) < 1e-9, k
