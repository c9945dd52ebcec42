"""CPU goldens for bench.py's own timed batch (build container only).

bench.py times config 2 on the 4096 seeded parameters of
``seeded_parameters(4096, seed=1000)``; its ``parity`` block compares the
device results of the first ``--n`` of them with

* the oracle (oracle/ddnm_oracle.py) -- x, lam, n_iter and whether every
  tol/Armijo decision on the trajectory cleared the merit noise floor
  ("robust", SURVEY.md §7 hard part 1);
* the reference itself (``ddrom.driver.solve_rom``, driver.py:554-597,
  compute_error=False) on the reference instance the committed artifacts were
  extracted from (artifacts_cache/c0_nm.pkl, tools/make_artifacts.py).

Output: tests/golden/bench_c0_parity.npz (small: n x (40 + 8) doubles).
"""

from __future__ import annotations

import argparse
import os
import pickle
import sys
from multiprocessing import get_context

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

REF = "/root/reference/pkg/src"


def _oracle(args):
    from oracle import ddnm_oracle as O
    path, mus = args
    inst = O.Instance(path)
    out = []
    for a, lam in mus:
        r = O.solve(inst, a, lam)
        robust = min(r.margins) > 1e-13 * r.merit_history[0]
        out.append((r.x, r.lam, r.n_iter, robust))
    return out


def _reference(args):
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import warnings

    from ddrom.burgers import ParameterPoint
    from ddrom.driver import solve_rom
    from ddrom.sqp import SqpConfig
    pkl, mus = args
    with open(pkl, "rb") as f:
        inst = pickle.load(f)
    out = []
    for a, lam in mus:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            sol, _ = solve_rom(inst, ParameterPoint(float(a), float(lam)), SqpConfig(),
                               compute_error=False)
        out.append((sol.sqp.x, sol.sqp.lam, sol.sqp.n_iter))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--name", default="c0_nm")
    a = ap.parse_args()
    from paper_2305_15163_b200.burgers import seeded_parameters
    mu = seeded_parameters(4096, seed=1000)[:a.n]
    path = os.path.join(ROOT, "tests", "golden", f"{a.name}_artifacts.npz")
    chunks = [mu[i::a.procs].tolist() for i in range(a.procs)]
    res = {"mu": mu}
    with get_context("fork").Pool(a.procs) as pool:
        parts = pool.map(_oracle, [(path, c) for c in chunks])
    rows = [None] * a.n
    for i, p in enumerate(parts):
        for j, r in enumerate(p):
            rows[i + j * a.procs] = r
    res["oracle_x"] = np.array([r[0] for r in rows])
    res["oracle_lam"] = np.array([r[1] for r in rows])
    res["oracle_n_iter"] = np.array([r[2] for r in rows], np.int64)
    res["robust"] = np.array([r[3] for r in rows], np.int64)
    pkl = os.path.join(ROOT, "artifacts_cache", f"{a.name}.pkl")
    if os.path.exists(pkl) and os.path.isdir(REF):
        with get_context("fork").Pool(a.procs) as pool:
            parts = pool.map(_reference, [(pkl, c) for c in chunks])
        rows = [None] * a.n
        for i, p in enumerate(parts):
            for j, r in enumerate(p):
                rows[i + j * a.procs] = r
        res["reference_x"] = np.array([r[0] for r in rows])
        res["reference_lam"] = np.array([r[1] for r in rows])
        res["reference_n_iter"] = np.array([r[2] for r in rows], np.int64)
        ex = max(float(np.max(np.abs(res["oracle_x"][k] - res["reference_x"][k]))
                       / np.max(np.abs(res["reference_x"][k])))
                 for k in range(a.n))
        print("oracle vs reference: max rel x", ex, "n_iter equal",
              int(np.sum(res["oracle_n_iter"] == res["reference_n_iter"])), "/", a.n)
    print("robust", int(res["robust"].sum()), "/", a.n)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "bench_c0_parity.npz"), **res)


if __name__ == "__main__":
    main()
