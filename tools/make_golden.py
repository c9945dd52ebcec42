"""Turn reference ROM instances into committed, reference-free fixtures.

Run in the build container only (imports the reference from
``/root/reference/pkg/src``; nothing on the GPU box reads it).  For every
instance pickled by ``tools/make_artifacts.py`` it writes

* ``tests/golden/<name>_artifacts.npz`` -- everything the online solve
  consumes, extracted exactly the way ``driver.build_problem`` builds it
  (driver.py:356-436): per block the decoder subnet (hyper.py:200-222) or the
  restricted POD basis (pod.py:95-97), the full interface decoder
  (autoencoder.py:104-112), the sampled residual rows and local column order
  of ``RestrictedResidual`` (driver.py:392-396), ``CA = C @ A_i``
  (driver.py:368-369), and the fitted RBF initializer (driver.py:59-90 with
  scipy's private ``_coeffs/_shift/_scale/powers``);
* ``tests/golden/<name>_golden.npz`` -- reference outputs on a seeded mu
  batch: ``init_guess`` (driver.py:442-458), the full ``solve_rom`` result
  (driver.py:554-597; x, lam, n_iter, merit/objective/alpha histories,
  failure), and for the first few mu the per-block ``eval_gradients`` pieces
  at (x0, lam0) (sqp.py:117-146), both decoders' values/Jacobians, the
  sampled boundary vectors, the dense restricted Jacobian and the first KKT
  step (sqp.py:162-208).
"""

from __future__ import annotations

import argparse
import json
import os
import pickle
import sys
import warnings

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def extract(inst, full_maps: bool = True) -> dict:
    """The package's own intake (paper_2305_15163_b200/intake.py)."""
    sys.path.insert(0, ROOT)
    from paper_2305_15163_b200.intake import arrays_from_ddrom
    return arrays_from_ddrom(inst, full_maps=full_maps)


def _golden_one(inst, mu, k, detail, dense_jd):
    """One mu of ``goldens`` (process-pool worker): batch rows as
    (index, value) pairs, detail arrays as-is."""
    sub = goldens(inst, 1, 0, 1 if detail else 0, mu=mu[k:k + 1], dense_jd=dense_jd)
    out = {}
    for key, v in sub.items():
        if key in ("mu", "seed"):
            continue
        if key.startswith("d0_"):
            out[f"d{k}_" + key[3:]] = v
        else:
            out[key] = (k, v[0])
    return out


def goldens(inst, B: int, seed: int, n_detail: int, mu=None, dense_jd: bool = True,
            procs: int = 1) -> dict:
    from ddrom.burgers import ParameterPoint, assemble
    from ddrom.driver import build_problem, init_guess, solve_rom
    from ddrom.errors import ConvergenceError
    from ddrom.hyper import extract_subnet, hr_rows_for_subdomain
    from ddrom.partition import RestrictedResidual
    from ddrom.sqp import SqpConfig, assemble_and_solve_kkt, eval_gradients

    cfg = SqpConfig()
    if mu is None:
        rng = np.random.default_rng(seed)
        a = rng.uniform(1.0, 1.0e4, B)
        lam = rng.uniform(5.0, 25.0, B)
        mu = np.stack([a, lam], axis=1)
    else:
        a, lam = mu[:, 0], mu[:, 1]
    n_D = sum(ni + ng for ni, ng in inst.latent_layout)
    n_C = inst.n_mult
    K = cfg.max_iter
    g = {
        "mu": mu, "seed": np.int64(seed),
        "x0": np.zeros((B, n_D)), "lam0": np.zeros((B, n_C)),
        "x": np.zeros((B, n_D)), "lam": np.zeros((B, n_C)),
        "n_iter": np.zeros(B, np.int64), "converged": np.zeros(B, np.int64),
        "failure": np.zeros(B, np.int64),           # 0 none, 1 line_search, 2 kkt
        "merit_hist": np.full((B, K + 1), np.nan),
        "obj_hist": np.full((B, K + 1), np.nan),
        "alpha_hist": np.full((B, K), np.nan),
    }
    part = inst.partition
    if procs > 1:
        from multiprocessing import get_context
        with get_context("fork").Pool(procs) as pool:
            parts = pool.starmap(_golden_one, [(inst, mu, k, k < n_detail, dense_jd)
                                               for k in range(B)], chunksize=1)
        for part_g in parts:
            for key, v in part_g.items():
                if isinstance(v, tuple):      # (row index, value) of a batch array
                    g[key][v[0]] = v[1]
                else:
                    g[key] = v
        return g
    for k in range(B):
        p = ParameterPoint(float(a[k]), float(lam[k]))
        ops = assemble(part.grid, p)
        prob = build_problem(inst, ops)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            x0, lam0 = init_guess(inst, p, ops=ops, prob=prob)
        g["x0"][k], g["lam0"][k] = x0, lam0
        try:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                sol, rec = solve_rom(inst, p, cfg, compute_error=False)
        except ConvergenceError:
            g["failure"][k] = 2
            continue
        r = sol.sqp
        g["x"][k], g["lam"][k] = r.x, r.lam
        g["n_iter"][k] = r.n_iter
        g["converged"][k] = int(r.converged)
        g["failure"][k] = 0 if r.failure_reason is None else 1
        g["merit_hist"][k, :len(r.merit_history)] = r.merit_history
        g["obj_hist"][k, :len(r.objective_history)] = r.objective_history
        g["alpha_hist"][k, :len(r.alpha_history)] = r.alpha_history
        if k < n_detail:
            ev = eval_gradients(prob, x0, lam0)
            g[f"d{k}_rho"] = ev.rho
            g[f"d{k}_con"] = ev.con
            g[f"d{k}_merit"] = np.float64(ev.merit)
            g[f"d{k}_objective"] = np.float64(ev.objective)
            s, s_lam = assemble_and_solve_kkt(prob, ev, cfg.reg_scale)
            g[f"d{k}_step"] = s
            g[f"d{k}_step_lam"] = s_lam
            for i, be in enumerate(ev.blocks):
                q = f"d{k}_b{i}_"
                g[q + "Br"] = be.Br
                g[q + "R_int"] = be.R_int
                g[q + "R_gam"] = be.R_gam
                g[q + "con_val"] = be.con_val
                g[q + "con_jac"] = be.con_jac
            for i, (xi, xg) in enumerate(inst.split_latent(x0)):
                q = f"d{k}_b{i}_"
                sub = part.subdomains[i]
                rows = inst.hr[i].apply_B_rows()
                io, gio = hr_rows_for_subdomain(part, i, rows)
                im, gm = inst.interior_maps[i], inst.interface_maps[i]
                srpc = inst.constraint_mode == "srpc"
                if hasattr(im, "restrict_outputs"):
                    si = im.restrict_outputs(io)
                else:
                    si = extract_subnet(im, io)
                if srpc and gio.size:
                    gm = (gm.restrict_outputs(gio) if hasattr(gm, "restrict_outputs")
                          else extract_subnet(gm, gio))
                g[q + "int_g"] = si.decode(xi)
                g[q + "int_J"] = np.asarray(si.jacobian(xi))
                if srpc and not gio.size:
                    g[q + "gam_g"] = np.zeros(0)
                    g[q + "gam_J"] = np.zeros((0, xg.size))
                else:
                    g[q + "gam_g"] = gm.decode(xg)
                    g[q + "gam_J"] = np.asarray(gm.jacobian(xg))
                cols = np.concatenate([sub.interior_cols[io],
                                       sub.interface_cols[gio]])
                rr = RestrictedResidual(ops, sub.res_rows[rows], cols)
                v = np.concatenate([g[q + "int_g"],
                                    g[q + "gam_g"] if srpc else g[q + "gam_g"][gio]])
                g[q + "stencil_r"] = rr.residual(v)
                if dense_jd:
                    g[q + "stencil_Jd"] = rr.jacobian(v).toarray()
                n = part.grid.nnode
                rws = sub.res_rows[rows]
                node = np.where(rws < n, rws, rws - n)
                isu = rws < n
                g[q + "bx"] = np.where(isu, ops.bux[node], ops.bvx[node])
                g[q + "by"] = np.where(isu, ops.buy[node], ops.bvy[node])
                g[q + "bc"] = np.where(isu, ops.cu[node], ops.cv[node])
    return g


def state_goldens(inst, g: dict, n: int) -> dict:
    """Reference ``instance.decode`` (driver.py:148-152) of the golden
    solutions, and ``relative_error`` (driver.py:496-507) against the
    monolithic FOM (``solve_monolithic``, the reference's compute_error path
    driver.py:566-569) for the first ``n`` mu."""
    from ddrom.burgers import ParameterPoint
    from ddrom.driver import relative_error, restrict_blocks
    from ddrom.burgers import solve_monolithic

    from ddrom.errors import ConvergenceError
    part = inst.partition
    rows = []
    out = {}
    for k in range(g["mu"].shape[0]):
        if len(rows) == n:
            break
        p = ParameterPoint(float(g["mu"][k, 0]), float(g["mu"][k, 1]))
        try:
            fom, _ = solve_monolithic(part.grid, p)
        except ConvergenceError:
            continue          # the FOM Newton stagnates at this mu: take the next one
        j = len(rows)
        states = inst.decode(g["x"][k])
        out[f"s{j}"] = np.concatenate([np.concatenate([xi, xg]) for xi, xg in states])
        out[f"fom{j}"] = np.asarray(fom, dtype=float)
        out[f"err{j}"] = np.float64(relative_error(restrict_blocks(part, fom), states))
        rows.append(k)
    out["mu"] = g["mu"][rows]
    out["x"] = g["x"][rows]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cache", default=os.path.join(ROOT, "artifacts_cache"))
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    ap.add_argument("--names", nargs="*",
                    default=["tiny_nm", "tiny_ls", "c0_nm", "c0_ls", "tiny_nmg", "tiny_srpc",
                             "tiny_lsg", "tiny_lss", "c0_nmg", "c0_srpc"])
    ap.add_argument("--B", type=int, default=16)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--detail", type=int, default=3)
    ap.add_argument("--states", type=int, default=3, help="mu with decoded-state goldens")
    ap.add_argument("--procs", type=int, default=1, help="mu solved in parallel")
    ap.add_argument("--big", action="store_true",
                    help="480^2 / 960^2 instances: no full maps, no dense Jd, no states")
    ap.add_argument("--artifacts-only", action="store_true",
                    help="rewrite the artifacts and state goldens, keep *_golden.npz")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    for name in a.names:
        with open(os.path.join(a.cache, f"{name}.pkl"), "rb") as f:
            inst = pickle.load(f)
        art = extract(inst, full_maps=not a.big)
        np.savez_compressed(os.path.join(a.out, f"{name}_artifacts.npz"), **art)
        gpath = os.path.join(a.out, f"{name}_golden.npz")
        if a.artifacts_only:
            gd = dict(np.load(gpath))
        else:
            gd = goldens(inst, a.B, a.seed, a.detail, dense_jd=not a.big, procs=a.procs)
            np.savez_compressed(gpath, **gd)
        if not a.big:
            st = state_goldens(inst, gd, a.states)
            np.savez_compressed(os.path.join(a.out, f"{name}_states.npz"), **st)
        print(name, "n_iter", gd["n_iter"].tolist(), "failure",
              gd["failure"].tolist(), flush=True)


if __name__ == "__main__":
    main()
