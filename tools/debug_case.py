"""Compare one mu's device trajectory with the oracle's (debug aid).

usage: python tools/debug_case.py <instance> <k> [slots]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2305_15163_b200 as P  # noqa: E402
from oracle import ddnm_oracle as O  # noqa: E402

name, k = sys.argv[1], int(sys.argv[2])
slots = int(sys.argv[3]) if len(sys.argv) > 3 else 0
path = os.path.join(ROOT, "tests", "golden", f"{name}_artifacts.npz")
g = dict(np.load(os.path.join(ROOT, "tests", "golden", f"{name}_golden.npz")))
inst, oi = P.RomInstance.load(path), O.Instance(path)
mu = g["mu"][k:k + 1]
res = P.solve_rom_batch(inst, mu, slots=slots)
r = O.solve(oi, *mu[0])
np.set_printoptions(precision=6, linewidth=150)
print("device: n_iter", res.n_iter[0], "status", res.status[0], "n_reg", res.n_reg[0],
      "n_evals", res.n_evals[0])
print("  merit", res.merit_hist[0, :res.n_iter[0] + 2])
print("  alpha", res.alpha_hist[0, :res.n_iter[0] + 1])
print("  |x|max", np.abs(res.x[0]).max(), "lam0 rel", np.abs(res.lam0[0] - g["lam0"][k]).max())
print("oracle: n_iter", r.n_iter, "failure", r.failure_reason, "n_evals", r.n_evals, "reg", r.n_regularized if hasattr(r, "n_regularized") else "?")
print("  merit", np.array(r.merit_history))
print("  alpha", np.array(r.alpha_history))
print("  |x|max", np.abs(r.x).max())
