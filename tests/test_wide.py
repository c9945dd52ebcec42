"""The batch-wide engine (one lane per mu, csrc/ddnm_wide.cu) against the
persistent slot kernels, the oracle and the reference goldens.

The default engine of solve_rom_batch is "auto" (wide when the instance is
eligible), so tests/test_gpu_parity.py already gates the wide engine against
the oracle and the reference on every NM / WFPC / collocation instance; this
module covers what is specific to it: the per-round packets against k_dd_eval,
agreement of the two engines, exactness of the speculative step lengths,
independence of the batch composition, eligibility and the C-ABI selectors."""

import numpy as np
import pytest

import paper_2305_15163_b200 as P
from paper_2305_15163_b200 import _native as N
from paper_2305_15163_b200.subdomain import DeviceRoundEngine

from .conftest import golden_path
from .test_oracle_golden import rel

pytestmark = pytest.mark.gpu

WIDE = ["tiny_nm", "c0_nm", "c3s_nm", "dd16_nm", "tiny42_nm", "c3_nm", "c4_nm"]
NOT_WIDE = ["tiny_ls", "c0_ls", "tiny_srpc", "tiny_nmg", "c0_lss"]


def lanes(B):
    return max(2 * ((B + 31) // 32 * 32), 1024)


@pytest.mark.parametrize("name", WIDE)
def test_packets_match_slot_kernels(name, gpu_instances):
    """One evaluation round at the initial points: the wide kernels' packets
    (Gram blocks, projections, constraint values and Jacobians, r^T r per
    block) equal k_dd_eval's to rounding (different summation orders)."""
    inst = gpu_instances[name]
    assert inst.context().info.wide == 1
    B = 8 if name in ("c3_nm", "c4_nm") else 40
    mu = P.seeded_parameters(B, seed=11)
    nb = inst.n_blocks
    pk = {}
    for wide in (False, True):
        eng = DeviceRoundEngine(inst)
        eng.begin(mu, P.SqpConfig(), None, None, 0, nb)
        stride = eng.packet_len(0, nb)
        if wide:
            eng.set_wide(True)
        rows = lanes(B) if wide else B
        packets = eng.buffer(rows * stride)
        eng.eval(packets, stride)
        eng.torch.cuda.synchronize()
        pk[wide] = packets.cpu().numpy().reshape(rows, stride)[:B].copy()
        eng.finish(mu)
    a, b = pk[False], pk[True]
    scale = np.abs(a).max(axis=0, keepdims=True)
    scale[scale == 0] = 1.0
    assert np.max(np.abs(a - b) / scale) < 1e-12


@pytest.mark.parametrize("name", ["tiny_nm", "c0_nm", "c3s_nm", "dd16_nm"])
def test_engines_agree(name, gpu_instances, goldens):
    """Both engines against the reference goldens (x, lambda 1e-9) and against
    each other: same decisions on evaluations that differ by rounding, so the
    iteration counts agree except where a decision sits in the round-off
    floor (same allowance as the oracle-vs-device gate)."""
    inst, g = gpu_instances[name], goldens[name]
    mu = g["mu"]
    rs = P.solve_rom_batch(inst, mu, engine="slots")
    rw = P.solve_rom_batch(inst, mu, engine="wide")
    assert rs.rounds == 0 and rs.launches == 1
    assert rw.rounds > 0 and rw.launches == 2 + 5 * rw.rounds
    # lanes launched (with the unused speculative candidates) vs evaluations consumed
    lanes = inst.context().lanes()
    assert int(rw.n_evals.sum()) <= lanes <= 2 * int(rw.n_evals.sum())
    for r in (rs, rw):
        for k in range(mu.shape[0]):
            assert rel(r.x[k], g["x"][k]) < 1e-9 and rel(r.lam[k], g["lam"][k]) < 1e-9
        assert r.counters[0] == int(r.n_evals.sum()) * inst.n_blocks
    same = int((rs.n_iter == rw.n_iter).sum())
    assert mu.shape[0] - same <= max(1, mu.shape[0] // 8), (name, same)
    np.testing.assert_allclose(rw.x0, rs.x0, rtol=1e-13, atol=0)
    np.testing.assert_allclose(rw.lam0, rs.lam0, rtol=1e-9, atol=1e-9 * np.abs(rs.lam0).max())


def test_speculative_step_lengths_are_exact(monkeypatch):
    """Evaluating a mu's next step lengths in the same round changes nothing:
    with and without speculation every output is bitwise the same -- and the
    rounds drop (a line-search failure costs 31 evaluations, sqp.py:275-293)."""
    mu = P.seeded_parameters(300, seed=1000)
    spec = P.solve_rom_batch(P.RomInstance.load(golden_path("c0_nm", "artifacts")), mu, engine="wide")
    monkeypatch.setenv("DDNM_WIDE_NOSPEC", "1")      # read when the context is created
    plain = P.solve_rom_batch(P.RomInstance.load(golden_path("c0_nm", "artifacts")), mu, engine="wide")
    for f in ("x", "lam", "n_iter", "n_evals", "status", "n_reg", "merit", "objective", "merit_hist",
              "obj_hist", "alpha_hist", "x0", "lam0"):
        np.testing.assert_array_equal(getattr(spec, f), getattr(plain, f), err_msg=f)
    assert np.any(spec.status == N.STATUS_LINE_SEARCH)       # the long backtracking runs are there
    assert plain.rounds >= int(plain.n_evals.max())      # one evaluation per mu per round
    assert spec.rounds < plain.rounds
    assert spec.counters == plain.counters                   # consumed evaluations only


@pytest.mark.parametrize("name", ["c0_nm", "tiny42_nm"])
def test_batch_composition_invariance_wide(name, gpu_instances):
    """A mu alone, in a sub-batch or in the batch: bitwise the same (lanes are
    independent; the partial sums of a mu do not depend on what else runs --
    neither on the item granularity of the round nor on its lane)."""
    inst = gpu_instances[name]
    mu = P.seeded_parameters(341, seed=5)
    full = P.solve_rom_batch(inst, mu, engine="wide")
    sub = P.solve_rom_batch(inst, mu[100:137], engine="wide")
    np.testing.assert_array_equal(sub.x, full.x[100:137])
    np.testing.assert_array_equal(sub.lam, full.lam[100:137])
    np.testing.assert_array_equal(sub.n_evals, full.n_evals[100:137])
    for k in (0, 340):
        one = P.solve_rom_batch(inst, mu[k:k + 1], engine="wide")
        np.testing.assert_array_equal(one.x[0], full.x[k])
        np.testing.assert_array_equal(one.lam[0], full.lam[k])
        assert one.n_iter[0] == full.n_iter[k]
    again = P.solve_rom_batch(inst, mu, engine="wide")
    np.testing.assert_array_equal(again.x, full.x)


@pytest.mark.parametrize("name", ["c3_nm", "c4_nm"])
def test_big_configs_wide(name, gpu_instances, goldens):
    """BASELINE configs 3 (480^2) and 4 (960^2, 4x4) through the wide engine:
    the reference's solutions on every golden mu, and the reference's
    iteration counts."""
    inst, g = gpu_instances[name], goldens[name]
    res = P.solve_rom_batch(inst, g["mu"], engine="wide")
    for k in range(g["mu"].shape[0]):
        assert rel(res.x[k], g["x"][k]) < 1e-9 and rel(res.lam[k], g["lam"][k]) < 1e-9
    np.testing.assert_array_equal(res.n_iter, g["n_iter"])
    assert np.all(res.n_reg == 0)


@pytest.mark.parametrize("name", NOT_WIDE)
def test_ineligible_instances_use_the_slot_kernels(name, gpu_instances):
    """Linear maps, SRPC coupling and gappy HR are not built for the wide
    engine: auto runs the persistent kernel, asking for wide fails loudly."""
    inst = gpu_instances[name]
    assert inst.context().info.wide == 0
    mu = P.seeded_parameters(4, seed=3)
    r = P.solve_rom_batch(inst, mu)
    assert r.rounds == 0
    with pytest.raises(NotImplementedError):         # DDNM_EUNSUPPORTED
        P.solve_rom_batch(inst, mu, engine="wide")
    with pytest.raises(ValueError):
        P.solve_rom_batch(inst, mu, engine="fast")
    eng = DeviceRoundEngine(inst)
    eng.begin(mu, P.SqpConfig(), None, None, 0, inst.n_blocks)
    with pytest.raises(NotImplementedError):
        eng.set_wide(True)
    eng.finish(mu)


def test_wide_needs_every_block(gpu_instances):
    """A rank of a subdomain-sharded solve owns a block range: no wide there."""
    inst = gpu_instances["dd16_nm"]
    mu = P.seeded_parameters(4, seed=3)
    eng = DeviceRoundEngine(inst)
    eng.begin(mu, P.SqpConfig(), None, None, 0, 8)
    with pytest.raises(NotImplementedError):
        eng.set_wide(True)
    eng.finish(mu)


def test_environment_selectors(gpu_instances, monkeypatch):
    inst = gpu_instances["tiny_nm"]
    mu = P.seeded_parameters(8, seed=2)
    assert P.solve_rom_batch(inst, mu).rounds > 0
    monkeypatch.setenv("DDNM_WIDE", "0")
    assert P.solve_rom_batch(inst, mu).rounds == 0
    assert P.solve_rom_batch(inst, mu, engine="wide").rounds > 0     # the explicit choice wins
    monkeypatch.delenv("DDNM_WIDE")
    monkeypatch.setenv("DDNM_WIDE_MIN_B", "9")
    assert P.solve_rom_batch(inst, mu).rounds == 0
    assert P.solve_rom_batch(inst, P.seeded_parameters(9, seed=2)).rounds > 0


def _exchange(ranks):
    """What the all-gathers of the trial records do between in-process ranks."""
    from .test_subdomain import _exchange_trials
    _exchange_trials(ranks)


@pytest.mark.parametrize("name,world", [("dd16_nm", 1), ("dd16_nm", 2), ("dd16_nm", 3), ("c0_nm", 2),
                                        ("c4_nm", 4)])
def test_sharded_ranks_with_wide_evaluation(name, world, gpu_instances):
    """Subdomain-sharded rounds whose ranks evaluate their blocks with the
    wide kernels (one packet per mu, any block range): a block's partial sums
    do not depend on which rank computes them, so every rank count reproduces
    the unsharded wide solve bit for bit (speculation changes nothing either)."""
    import torch

    from paper_2305_15163_b200.subdomain import ShardedSolve
    from .test_subdomain import _exchange_results
    inst = gpu_instances[name]
    B = 6 if name == "c4_nm" else 24
    mu = P.seeded_parameters(B, seed=4)
    ref = P.solve_rom_batch(inst, mu, engine="wide")
    cfg = P.SqpConfig()
    ranks = [ShardedSolve(inst, mu, cfg, r, world) for r in range(world)]
    assert all(sh.wide for sh in ranks)
    gathered = torch.empty(world * ranks[0].B * ranks[0].stride, dtype=torch.float64, device="cuda")
    active = ranks[0].active
    while active:
        parts = [sh.eval().clone() for sh in ranks]
        torch.cat(parts, out=gathered)
        active = sum(sh.step(gathered) for sh in ranks)
        _exchange(ranks)
    _exchange_results(ranks)
    for sh in ranks:
        r = sh.result(group=False)
        for k in ("x", "lam", "n_iter", "n_evals", "status", "merit"):
            np.testing.assert_array_equal(getattr(r, k), getattr(ref, k), err_msg=k)


def test_sharded_driver_uses_wide_by_default(gpu_instances, goldens):
    """solve_rom_batch_subdomain_sharded at one rank: wide evaluation when the
    instance has it (bitwise the wide engine's solve), k_dd_eval on request or
    for the peer-store transport; the reference goldens either way."""
    inst, g = gpu_instances["dd16_nm"], goldens["dd16_nm"]
    mu = g["mu"]
    ref = P.solve_rom_batch(inst, mu, engine="wide")
    res = P.solve_rom_batch_subdomain_sharded(inst, mu)
    np.testing.assert_array_equal(res.x, ref.x)
    np.testing.assert_array_equal(res.n_evals, ref.n_evals)
    assert res.counters[0] == int(res.n_evals.sum()) * inst.n_blocks
    slots = P.solve_rom_batch_subdomain_sharded(inst, mu, wide=False)
    for r in (res, slots):
        for k in range(mu.shape[0]):
            assert rel(r.x[k], g["x"][k]) < 1e-9 and rel(r.lam[k], g["lam"][k]) < 1e-9
    with pytest.raises(ValueError):
        P.solve_rom_batch_subdomain_sharded(inst, mu, transport="p2p", wide=True)
