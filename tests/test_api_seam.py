"""The drop-in seam: the package's online API mirrors the reference's
(``ddrom.driver`` / ``ddrom.sqp``) signatures, defaults and record types,
and ``RomInstance.from_ddrom`` takes the reference's own instance.

CPU only; compares against /root/reference when it is present (the build
container) and skips otherwise (the GPU box has no reference)."""

import inspect
import os
import sys

import numpy as np
import pytest

import paper_2305_15163_b200 as P

REF = "/root/reference/pkg/src"
needs_ref = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import ddrom.driver as D
    import ddrom.sqp as S
    return D, S


def _params(fn):
    return [(p.name, p.kind, p.default) for p in inspect.signature(fn).parameters.values()]


@needs_ref
@pytest.mark.parametrize("name", ["solve_rom", "init_guess", "build_problem"])
def test_driver_signatures_match(name):
    D, _ = _ref()
    ours, ref = _params(getattr(P, name)), _params(getattr(D, name))
    assert [(n, k) for n, k, _ in ours] == [(n, k) for n, k, _ in ref]
    for (n, _, d1), (_, _, d2) in zip(ours, ref):
        if d2 is inspect.Parameter.empty or isinstance(d2, (int, float, str, bool, type(None))):
            assert d1 == d2 or (isinstance(d2, float) and np.isnan(d2) and np.isnan(d1)), n


@needs_ref
def test_sqp_signatures_match():
    _, S = _ref()
    assert [n for n, _, _ in _params(P.iterate)] == [n for n, _, _ in _params(S.iterate)]
    ref_cfg, ours = S.SqpConfig(), P.SqpConfig()
    for f in ("tol", "max_iter", "armijo_c1", "backtrack_factor", "max_halvings", "reg_scale"):
        assert getattr(ours, f) == getattr(ref_cfg, f), f


@needs_ref
def test_record_types_match():
    D, _ = _ref()
    import dataclasses
    assert [f.name for f in dataclasses.fields(P.BenchmarkRecord)] == \
        [f.name for f in dataclasses.fields(D.BenchmarkRecord)]
    assert P.BenchmarkRecord.HEADER == D.BenchmarkRecord.HEADER
    assert [f.name for f in dataclasses.fields(P.RomSolution)] == \
        [f.name for f in dataclasses.fields(D.RomSolution)]
    r = P.BenchmarkRecord(label="x", config={"rom": "nmrom"}, a=1.0, lam=5.0)
    assert len(r.row()) == len(r.HEADER)


@needs_ref
def test_reference_ops_accepted():
    """build_problem/init_guess take the reference's FomOperators (they read
    ``param``) as well as ours."""
    from ddrom.burgers import Grid2D, ParameterPoint, assemble
    from paper_2305_15163_b200.driver import _param_of
    ops = assemble(Grid2D(8, 8, 0.1), ParameterPoint(100.0, 10.0))
    assert _param_of(ops) == P.ParameterPoint(100.0, 10.0)
    assert _param_of(P.assemble(P.Grid2D(8, 8), P.ParameterPoint(3.0, 7.0))).a == 3.0


@needs_ref
def test_from_ddrom_intake_matches_reference_eval(tmp_path):
    """A small reference instance built by the reference itself goes through
    RomInstance.from_ddrom; the oracle evaluated on the extracted arrays
    reproduces the reference's own eval_gradients (sqp.py:117-146) at a
    point -- the intake keeps everything build_problem uses."""
    import warnings
    _ref()
    from dataclasses import replace

    from ddrom.autoencoder import TrainConfig
    from ddrom.burgers import Grid2D, ParameterPoint, assemble
    from ddrom.driver import attach_hr, build_nmrom, build_problem, fit_initializer
    from ddrom.partition import build_partition
    from ddrom.snapshots import generate, sample_grid
    from ddrom.sqp import eval_gradients

    from oracle import ddnm_oracle as O
    grid = Grid2D(12, 12, 0.1)
    part = build_partition(grid, 2, 2)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        snap = generate(grid, sample_grid(3, 3), part, tol=1e-7)
        nm = build_nmrom(part, snap, 3, 2, "wfpc", band=3, shift=1,
                         train_cfg=replace(TrainConfig(epochs=3), seed=0), wfpc_seed=0, n_c=2)
        inst = fit_initializer(attach_hr(nm, snap, "collocation", n_samples=20), snap)
    ours = P.RomInstance.from_ddrom(inst)
    assert ours.n_blocks == 4 and ours.n_mult == 2 and ours.has_full_decoders
    oi = O.Instance(ours.arrays)
    p = ParameterPoint(3000.0, 12.0)
    x = inst.initializer.query(p)
    lam = np.linspace(-1.0, 1.0, 2)
    ref = eval_gradients(build_problem(inst, assemble(grid, p)), x, lam)
    ev = O.eval_gradients(oi, oi.boundary(p.a, p.lam), x, lam)
    np.testing.assert_allclose(ev.rho, ref.rho, rtol=1e-12, atol=1e-12 * np.abs(ref.rho).max())
    np.testing.assert_allclose(ev.con, ref.con, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(O.rbf_query(oi, p.a, p.lam), x, rtol=1e-13)
