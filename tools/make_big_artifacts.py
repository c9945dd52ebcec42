"""Build the BASELINE config-3 (480^2) and config-4 (960^2) ROM instances with
the *reference* package (offline; build container only).

SURVEY.md §8(d1):

    config 3: Grid2D(480, 480, 0.1), 2x2 subdomains, sample_grid(8, 8),
              n = (8, 5), band 8, shift 1, 2% collocation rows (2304 per
              subdomain), n_C = 10, snapshots at tol 1e-4
    config 4: Grid2D(960, 960, 0.1), 4x4 subdomains, same nets/HR, n_C = 40,
              snapshots at tol 1e-3

Everything is a reference call; what differs from one sequential
``build_nmrom``/``attach_hr``/``fit_initializer`` chain is only how the work
is spread over the 8 host cores, and two recorded choices:

* snapshots: ``snapshots.generate`` (snapshots.py:103-160) is run once per
  a-row of the 8x8 grid (8 lam values, lam fastest, warm-started within the
  row) in 8 processes and the 8 ``SnapshotSet``s are concatenated in grid
  order.  A single ``generate`` call would warm-start each row's first point
  from the previous row's last one; here it starts cold (zeros), which
  changes only Newton's path to the same tolerance.
* ``--ordering``: the fill-reducing column ordering SuperLU uses inside the
  reference's Newton (``burgers.py:303``, default COLAMD).  960^2 uses
  MMD_AT_PLUS_A (half the fill, measured at 480^2: 60M vs 88M nonzeros), so
  8 factorizations fit in host memory at once.  Same Newton iteration, same
  tolerance; only the LU's round-off differs.
* training epochs are cut (``--epochs``, default 150; the reference default
  is 2000, ~2.7 h per 115k-output net).  The hot path's parity does not
  depend on how well the nets are trained: oracle, reference goldens and the
  device all consume the same trained weights.

The nets are trained in a process pool with exactly the seeds and arguments
``driver.train_nets`` uses (driver.py:234-246); the HR operators are built per
subdomain exactly as ``attach_hr`` does (driver.py:283-301), in a pool.
Output: ``artifacts_cache/<tag>_nm.pkl`` (git-ignored), consumed by
``tools/make_golden.py``.
"""

from __future__ import annotations

import argparse
import os
import pickle
import sys
import time
from multiprocessing import get_context

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import numpy as np  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_artifacts import _train_one  # noqa: E402

_ORDER = {"spec": "COLAMD"}


def _patch_ordering(spec: str):
    import scipy.sparse.linalg as spla
    from ddrom import burgers
    if spec == "COLAMD":
        return
    orig = spla.splu

    class _Spla:
        def __getattr__(self, k):
            return getattr(spla, k)

        @staticmethod
        def splu(A, **kw):
            kw.setdefault("permc_spec", spec)
            return orig(A, **kw)

    burgers.spla = _Spla()


def _gen_row(args):
    nx, ny, sx, sy, params, tol, spec = args
    _patch_ordering(spec)
    from ddrom.burgers import Grid2D
    from ddrom.partition import build_partition
    from ddrom.snapshots import generate
    grid = Grid2D(nx, ny, 0.1)
    part = build_partition(grid, sx, sy)
    t0 = time.time()
    snap = generate(grid, params, part, tol=tol)
    print(f"  row a={params[0].a:.1f}: {snap.n_mu} ok, {len(snap.failures)} failed, "
          f"iters {snap.newton_iters}, {time.time() - t0:.0f}s", flush=True)
    return snap


def _hr_one(args):
    from ddrom.hyper import greedy_sample, hr_collocation
    from ddrom.pod import pod
    R, n_samples, n_res, energy = args
    t0 = time.time()
    basis = pod(R, tol=energy).Phi                      # driver.py:294
    ns = min(max(n_samples, basis.shape[1]), n_res)     # driver.py:295
    rows = greedy_sample(basis, ns)                     # driver.py:296
    print(f"  hr: basis {basis.shape}, {ns} rows, {time.time() - t0:.0f}s", flush=True)
    return hr_collocation(rows, n_res)                  # driver.py:297


def merge(parts, grid, part):
    from ddrom.snapshots import SnapshotSet
    states = np.column_stack([p.states for p in parts])
    interior = {i: states[s.interior_cols, :] for i, s in enumerate(part.subdomains)}
    interface = {i: states[s.interface_cols, :] for i, s in enumerate(part.subdomains)}
    port = {}
    for pt in part.ports.ports:
        i = pt.members[0]
        pos = part.ports.member_positions(pt.index, i)
        port[pt.index] = interface[i][pos, :]
    residual = {i: np.column_stack([p.residual[i] for p in parts])
                for i in range(len(part.subdomains))}
    out = SnapshotSet(grid=grid, nsub_x=part.nsub_x, nsub_y=part.nsub_y,
                      params=[q for p in parts for q in p.params], states=states,
                      interior=interior, interface=interface, port=port,
                      residual=residual,
                      failures=[f for p in parts for f in p.failures],
                      newton_iters=[k for p in parts for k in p.newton_iters])
    out.check_port_consistency(part)
    return out


def build(tag, nx, sx, grid_n, tol, n_int, n_gam, n_c, n_samples, epochs,
          spec, procs, out, train_procs):
    from ddrom.burgers import Grid2D
    from ddrom.driver import (RomInstance, _wfpc_matrix_for, fit_initializer,
                              replace_instance)
    from ddrom.partition import build_partition
    from ddrom.snapshots import sample_grid

    os.makedirs(out, exist_ok=True)
    grid = Grid2D(nx, nx, 0.1)
    part = build_partition(grid, sx, sx)
    t0 = time.time()
    snap_path = os.path.join(out, f"{tag}_snap.pkl")
    if os.path.exists(snap_path):
        with open(snap_path, "rb") as f:
            snap = pickle.load(f)
    else:
        params = sample_grid(grid_n, grid_n)
        rows = [params[k * grid_n:(k + 1) * grid_n] for k in range(grid_n)]
        with get_context("fork").Pool(min(procs, grid_n)) as pool:
            parts = pool.map(_gen_row, [(nx, nx, sx, sx, r, tol, spec) for r in rows])
        snap = merge(parts, grid, part)
        with open(snap_path, "wb") as f:
            pickle.dump(snap, f, protocol=4)
    print(f"[{tag}] snapshots: {snap.n_mu} ok, {len(snap.failures)} failed, "
          f"{sum(r.shape[1] for r in snap.residual.values()) // len(snap.residual)} "
          f"residual columns per subdomain, {time.time() - t0:.0f}s", flush=True)

    nsub = len(part.subdomains)
    nets_path = os.path.join(out, f"{tag}_nets.pkl")
    if os.path.exists(nets_path):
        with open(nets_path, "rb") as f:
            nets_int, nets_gam = pickle.load(f)
    else:
        jobs = ([(snap.interior[i], n_int, "swish", 100 + i, 8, 1, epochs, 0)
                 for i in range(nsub)]
                + [(snap.interface[i], n_gam, "swish", 200 + i, 8, 1, epochs, 0)
                   for i in range(nsub)])
        t1 = time.time()
        with get_context("fork").Pool(min(train_procs, len(jobs))) as pool:
            res = pool.map(_train_one, jobs, chunksize=1)
        for k, (_, dt, best, ran) in enumerate(res):
            print(f"[{tag}] net {k}: {dt:.0f}s, best epoch {best}, ran {ran}", flush=True)
        nets_int = [r[0] for r in res[:nsub]]
        nets_gam = [r[0] for r in res[nsub:]]
        with open(nets_path, "wb") as f:
            pickle.dump((nets_int, nets_gam), f, protocol=4)
        print(f"[{tag}] training {time.time() - t1:.0f}s", flush=True)

    A, C = _wfpc_matrix_for(part, n_gam, n_c, 0)
    prov = {"rom": "nmrom", "constraint": "wfpc", "hr": "none",
            "n_int": n_int, "n_gam": n_gam, "seed": 0}
    nm = RomInstance(partition=part, interior_maps=nets_int,
                     interface_maps=nets_gam, constraint_mode="wfpc",
                     fom_constraints=A, wfpc_C=C, provenance=prov)
    t2 = time.time()
    with get_context("fork").Pool(min(procs, nsub)) as pool:
        ops = pool.map(_hr_one, [(snap.residual[i], n_samples, s.n_res, 1e-10)
                                 for i, s in enumerate(part.subdomains)], chunksize=1)
    nm = replace_instance(nm, hr=ops, provenance={**nm.provenance, "hr": "collocation",
                                                  "hr_samples": n_samples})
    print(f"[{tag}] hr {time.time() - t2:.0f}s", flush=True)
    nm = fit_initializer(nm, snap)
    nm.provenance["epochs"] = epochs
    nm.provenance["snap_tol"] = tol
    nm.provenance["splu_ordering"] = spec
    with open(os.path.join(out, f"{tag}_nm.pkl"), "wb") as f:
        pickle.dump(nm, f, protocol=4)
    print(f"[{tag}] done in {time.time() - t0:.0f}s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=["c3", "c4"], required=True)
    ap.add_argument("--out", default=os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "artifacts_cache"))
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--train-procs", type=int, default=os.cpu_count())
    ap.add_argument("--epochs", type=int, default=150)
    ap.add_argument("--ordering", default=None)
    a = ap.parse_args()
    if a.config == "c3":
        build("c3", 480, 2, 8, 1e-4, 8, 5, 10, 2304, a.epochs,
              a.ordering or "COLAMD", a.procs, a.out, a.train_procs)
    else:
        build("c4", 960, 4, 8, 1e-3, 8, 5, 40, 2304, a.epochs,
              a.ordering or "MMD_AT_PLUS_A", a.procs, a.out, a.train_procs)


if __name__ == "__main__":
    main()
