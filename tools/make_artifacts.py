"""Build the config-0/1 ROM instances with the *reference* package (offline).

This is test infrastructure, run once in the build container (where
``/root/reference`` exists).  It reproduces SURVEY.md §8(d1):

    grid = Grid2D(60, 60, 0.1); part = build_partition(grid, 2, 2)
    snap = generate(grid, sample_grid(6, 6), part, tol=1e-7)            (R8)
    nm   = build_nmrom(part, snap, 6, 4, "wfpc", band=8, shift=1,
                       train_cfg=TrainConfig(epochs=2000, seed=0),
                       wfpc_seed=0, n_c=8)                              (R4-R6)
    hr   = fit_initializer(attach_hr(nm, snap, "collocation",
                                     n_samples=180, energy=1e-10), snap) (R7)
    ls   = build_lsrom(part, snap, 20, 8, "wfpc", n_c=16) + same HR

The eight nets are trained in a process pool with exactly the seeds and
arguments ``driver.train_nets`` uses (driver.py:234-246), so the result is
identical to the sequential ``build_nmrom`` call; ``RomInstance`` is then
assembled exactly as ``build_nmrom`` does (driver.py:266-272).

Output: pickled reference instances under ``--out`` (default
``artifacts_cache/``, git-ignored).  ``tools/make_golden.py`` turns them into
the committed, reference-free fixtures the GPU box reads.
"""

from __future__ import annotations

import argparse
import os
import pickle
import sys
import time
from dataclasses import replace
from multiprocessing import get_context

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import numpy as np  # noqa: E402


def _train_one(args):
    from ddrom.autoencoder import TrainConfig, build_mask, train
    X, n, tag, offset, band, shift, epochs, seed = args
    cfg = replace(TrainConfig(epochs=epochs, seed=seed), seed=seed + offset)
    n_eff = max(1, min(n, X.shape[0] - 1))
    t0 = time.time()
    ae, hist = train(X, build_mask(X.shape[0], band, shift), n_eff, cfg,
                     activation=tag)
    return ae, time.time() - t0, hist["best_epoch"], len(hist["val_loss"])


def build(nx: int, ny: int, sx: int, sy: int, grid_n: int, snap_tol: float,
          n_int: int, n_gam: int, band: int, shift: int, epochs: int,
          n_c_nm: int, n_c_ls: int, n_samples: int, ls_dims, out: str,
          procs: int, tag: str):
    from ddrom.burgers import Grid2D
    from ddrom.driver import (RomInstance, _wfpc_matrix_for, attach_hr,
                              build_lsrom, fit_initializer)
    from ddrom.partition import build_partition
    from ddrom.snapshots import generate, sample_grid

    os.makedirs(out, exist_ok=True)
    t0 = time.time()
    grid = Grid2D(nx, ny, 0.1)
    part = build_partition(grid, sx, sy)
    snap_path = os.path.join(out, f"{tag}_snap.pkl")
    if os.path.exists(snap_path):
        with open(snap_path, "rb") as f:
            snap = pickle.load(f)
    else:
        snap = generate(grid, sample_grid(grid_n, grid_n), part, tol=snap_tol)
        with open(snap_path, "wb") as f:
            pickle.dump(snap, f)
    print(f"[{tag}] snapshots: {snap.n_mu} ok, {len(snap.failures)} failed, "
          f"{time.time() - t0:.1f}s", flush=True)

    nsub = len(part.subdomains)
    jobs = ([(snap.interior[i], n_int, "swish", 100 + i, band, shift, epochs, 0)
             for i in range(nsub)]
            + [(snap.interface[i], n_gam, "swish", 200 + i, band, shift,
                epochs, 0) for i in range(nsub)])
    t1 = time.time()
    with get_context("fork").Pool(min(procs, len(jobs))) as pool:
        res = pool.map(_train_one, jobs)
    for k, (_, dt, best, ran) in enumerate(res):
        print(f"[{tag}] net {k}: {dt:.1f}s, best epoch {best}, ran {ran}",
              flush=True)
    nets_int = [r[0] for r in res[:nsub]]
    nets_gam = [r[0] for r in res[nsub:]]
    print(f"[{tag}] training {time.time() - t1:.1f}s", flush=True)

    A, C = _wfpc_matrix_for(part, n_gam, n_c_nm, 0)
    prov = {"rom": "nmrom", "constraint": "wfpc", "hr": "none",
            "n_int": n_int, "n_gam": n_gam, "seed": 0}
    nm = RomInstance(partition=part, interior_maps=nets_int,
                     interface_maps=nets_gam, constraint_mode="wfpc",
                     fom_constraints=A, wfpc_C=C, provenance=prov)
    nm = fit_initializer(attach_hr(nm, snap, "collocation",
                                   n_samples=n_samples, energy=1e-10), snap)
    with open(os.path.join(out, f"{tag}_nm.pkl"), "wb") as f:
        pickle.dump(nm, f)
    if ls_dims is not None:
        ls = build_lsrom(part, snap, ls_dims[0], ls_dims[1], "wfpc",
                         n_c=n_c_ls)
        ls = fit_initializer(attach_hr(ls, snap, "collocation",
                                       n_samples=n_samples, energy=1e-10),
                             snap)
        with open(os.path.join(out, f"{tag}_ls.pkl"), "wb") as f:
            pickle.dump(ls, f)
    print(f"[{tag}] done in {time.time() - t0:.1f}s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c0", choices=["c0", "tiny", "dd16", "c3", "c3s", "tiny42"])
    ap.add_argument("--out", default=os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
        "artifacts_cache"))
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--epochs", type=int, default=None)
    a = ap.parse_args()
    if a.config == "c0":
        # SURVEY.md §8(d1) config 0 (NM) + config 1 (LS) on the same snapshots
        build(60, 60, 2, 2, 6, 1e-7, 6, 4, 8, 1, a.epochs or 2000, 8, 16,
              180, (20, 8), a.out, a.procs, "c0")
    elif a.config == "c3":
        # 480x480, 2x2, 8x8 mu grid, n = (8, 5),
        # band 8, 2% collocation rows (2304 per subdomain), n_C = 10
        build(480, 480, 2, 2, 8, 1e-7, 8, 5, 8, 1, a.epochs or 2000, 10, 10,
              2304, None, a.out, a.procs, "c3")
    elif a.config == "c3s":
        # config 3's layout at 120x120 (the reference's FOM Newton stagnates
        # at |r| ~ 1e-6 > tol = 1e-7 from 240x240 up, measured): 2x2, 8x8 mu
        # grid, n = (8, 5), band 8, 2% collocation rows (144), n_C = 10
        build(120, 120, 2, 2, 8, 1e-7, 8, 5, 8, 1, a.epochs or 2000, 10, 10,
              144, None, a.out, a.procs, "c3s")
    elif a.config == "dd16":
        # many-subdomain instance for subdomain sharding (config 4's layout at
        # a trainable size): 60x60 grid, 4x4 subdomains, n = (8, 5) and
        # n_C = 40 as config 4, 8x8 mu grid, 10% collocation rows
        build(60, 60, 4, 4, 8, 1e-7, 8, 5, 8, 1, a.epochs or 2000, 40, 40,
              45, None, a.out, a.procs, "dd16")
    elif a.config == "tiny42":
        # a latent pair outside the hand-written kernel list (the paper's
        # latent sweep starts at (4, 2)): 24x24, 2x2,
        # n = (4, 2), n_C = sum n_gam / 2 = 4
        build(24, 24, 2, 2, 4, 1e-7, 4, 2, 4, 1, a.epochs or 2000, 4, 4,
              40, None, a.out, a.procs, "tiny42")
    else:
        # small fast instance for CPU unit tests: 24x24 grid, 2x2 subdomains
        build(24, 24, 2, 2, 4, 1e-7, 4, 3, 4, 1, a.epochs or 2000, 4, 8,
              40, (8, 4), a.out, a.procs, "tiny")


if __name__ == "__main__":
    main()
