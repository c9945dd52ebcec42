"""Full decode of the SQP solutions (RomInstance.decode, driver.py:148-152)
and relative_error against a FOM state (driver.py:496-507).

The goldens (tests/golden/*_states.npz, tools/make_golden.py) hold the
reference's own ``instance.decode`` of its solutions and ``relative_error``
against its monolithic FOM solve (``solve_monolithic``) for three mu."""

import numpy as np
import pytest

from tests.conftest import ALL, BIG, golden_path

# the 480^2 / 960^2 instances carry no full maps (decode is off their solve path)
DEC = [n for n in ALL if n not in BIG]


def _states(name):
    return dict(np.load(golden_path(name, "states")))


def _flat(blocks):
    return np.concatenate([np.concatenate(p) for p in blocks])


# -- CPU: oracle pinned to the reference, host-side index helpers ---------------

@pytest.mark.parametrize("name", DEC)
def test_oracle_decode_matches_reference(name, oracle_instances):
    from oracle import ddnm_oracle as O
    inst, s = oracle_instances[name], _states(name)
    for k in range(s["x"].shape[0]):
        st = inst.decode(s["x"][k])
        np.testing.assert_array_equal(_flat(st), s[f"s{k}"])
        e = O.relative_error(inst.restrict_blocks(s[f"fom{k}"]), st)
        assert e == float(s[f"err{k}"])


def test_oracle_relative_error_rejects_zero_block(oracle_instances):
    from oracle import ddnm_oracle as O
    inst = oracle_instances["tiny_nm"]
    s = _states("tiny_nm")
    st = inst.decode(s["x"][0])
    with pytest.raises(ValueError):
        O.relative_error(inst.restrict_blocks(np.zeros_like(s["fom0"])), st)


@pytest.mark.parametrize("name", ["tiny_nm", "c0_ls"])
def test_restrict_and_assemble_host_helpers(name, oracle_instances):
    import paper_2305_15163_b200 as P
    inst = P.RomInstance.load(golden_path(name, "artifacts"))
    s = _states(name)
    fom = s["fom0"]
    got = inst.restrict_blocks(fom)
    ref = oracle_instances[name].restrict_blocks(fom)
    for (a, b), (c, d) in zip(got, ref):
        np.testing.assert_array_equal(a, c)
        np.testing.assert_array_equal(b, d)
    # every dof is held by some block, so merging the restriction is exact
    np.testing.assert_array_equal(inst.assemble_global(got), fom)
    assert [a.size + b.size for a, b in got] == [a + b for a, b in inst.state_layout]
    with pytest.raises(ValueError):
        inst.restrict_blocks(fom[:-1])


# -- GPU: device decode ----------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", DEC)
def test_decode_matches_reference_golden(name, gpu_instances):
    import paper_2305_15163_b200 as P
    inst, s = gpu_instances[name], _states(name)
    n = s["x"].shape[0]
    fom = np.stack([s[f"fom{k}"] for k in range(n)])
    dec = P.decode_batch(inst, s["x"], fom_states=fom)
    for k in range(n):
        ref = s[f"s{k}"]
        # swish/expit via the device exp (<= 2 ulp), sums in the reference order
        np.testing.assert_allclose(dec.states[k], ref, rtol=1e-12,
                                   atol=1e-13 * np.abs(ref).max())
        assert abs(dec.error[k] - float(s[f"err{k}"])) <= 1e-12 * float(s[f"err{k}"])
        for (a, b), (c, d) in zip(dec.blocks(k), inst.restrict_blocks(np.zeros(fom.shape[1]))):
            assert a.shape == c.shape and b.shape == d.shape


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c0_nm", "c0_ls"])
def test_decode_batch_of_solutions_matches_oracle(name, gpu_instances, oracle_instances):
    """Decode of a whole solved batch (ragged tile: B = 37) against the oracle."""
    import paper_2305_15163_b200 as P
    inst, oinst = gpu_instances[name], oracle_instances[name]
    res = P.solve_rom_batch(inst, P.seeded_parameters(37, seed=5))
    dec = P.decode_batch(inst, res.x)
    for k in (0, 7, 8, 36):
        ref = _flat(oinst.decode(res.x[k]))
        np.testing.assert_allclose(dec.states[k], ref, rtol=1e-12,
                                   atol=1e-13 * np.abs(ref).max())


@pytest.mark.gpu
def test_solve_rom_returns_states_and_error(gpu_instances, oracle_instances):
    import paper_2305_15163_b200 as P
    from oracle import ddnm_oracle as O
    inst, oinst = gpu_instances["c0_nm"], oracle_instances["c0_nm"]
    s = _states("c0_nm")
    p = P.ParameterPoint(*s["mu"][1])
    sol, rec = P.solve_rom(inst, p, fom_state=s["fom1"])
    ref = oinst.decode(sol.x_latent)
    for (a, b), (c, d) in zip(sol.states, ref):
        np.testing.assert_allclose(a, c, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(b, d, rtol=1e-12, atol=1e-13)
    e = O.relative_error(oinst.restrict_blocks(s["fom1"]), ref)
    assert abs(sol.error - e) <= 1e-12 * e and rec.error == sol.error
    # the device solution is the reference's to 1e-9, so is its error
    assert abs(sol.error - float(s["err1"])) <= 1e-6 * float(s["err1"])
    # the reference's default (compute_error=True, no fom_state): the FOM is
    # solved first (host, burgers.solve_monolithic semantics), then the error
    sol2, rec2 = P.solve_rom(inst, p)
    assert abs(sol2.error - float(s["err1"])) <= 1e-6 * float(s["err1"])
    assert rec2.fom_seconds > 0 and rec2.speedup == rec2.fom_seconds / rec2.parallel_seconds
    assert len(rec2.row()) == len(P.BenchmarkRecord.HEADER)
    _, rec3 = P.solve_rom(inst, p, compute_error=False)
    assert np.isnan(rec3.error) and np.isnan(rec3.fom_seconds)


@pytest.mark.gpu
def test_decode_edge_cases(gpu_instances):
    import paper_2305_15163_b200 as P
    inst = gpu_instances["tiny_nm"]
    s = _states("tiny_nm")
    empty = P.decode_batch(inst, np.zeros((0, inst.n_primal)))
    assert empty.states.shape == (0, sum(a + b for a, b in inst.state_layout))
    with pytest.raises(ValueError):
        P.decode_batch(inst, s["x"][:1], fom_states=np.zeros((1, s["fom0"].size)))
    with pytest.raises(ValueError):
        P.decode_batch(inst, np.zeros((2, inst.n_primal + 1)))
    # errors only (no states kept)
    d = P.decode_batch(inst, s["x"][:1], fom_states=s["fom0"][None], keep_states=False)
    assert d.states is None and abs(d.error[0] - float(s["err0"])) <= 1e-12 * float(s["err0"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c0_nm", "c3s_nm"])
def test_solve_subnet_rows_match_decode_rows(name, gpu_instances, goldens):
    """SURVEY §4's invariant between the two device decoders: the HR subnet
    rows the solve kernel evaluates (ddnm_eval_batch: interior outputs `io`)
    equal the full interior decoder's rows at those positions (k_decode,
    RomInstance.decode) -- to rounding, since the solve kernel contracts
    differently (fma, split-lane row sums; see ddnm_solve.cuh phase A/B)
    while k_decode keeps the reference's order."""
    import paper_2305_15163_b200 as P
    inst, g = gpu_instances[name], goldens[name]
    x = g["x"][:4]
    ev = P.eval_gradients_batch(inst, g["mu"][:4], x, g["lam"][:4], step=False)
    dec = P.decode_batch(inst, x)
    for k in range(4):
        for b, (xi, xg) in enumerate(dec.blocks(k)):
            io = inst.arrays[f"b{b}_io"]
            sub = ev.block(k, b)["int_g"]
            assert np.max(np.abs(sub - xi[io])) <= 1e-14 * max(np.max(np.abs(xi[io])), 1e-300)
