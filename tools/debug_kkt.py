"""Device vs oracle KKT solves along the oracle's trajectory (debug aid).

usage: python tools/debug_kkt.py <instance> <k> [n_steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2305_15163_b200 as P  # noqa: E402
from oracle import ddnm_oracle as O  # noqa: E402

name, k = sys.argv[1], int(sys.argv[2])
nst = int(sys.argv[3]) if len(sys.argv) > 3 else 4
path = os.path.join(ROOT, "tests", "golden", f"{name}_artifacts.npz")
g = dict(np.load(os.path.join(ROOT, "tests", "golden", f"{name}_golden.npz")))
inst, oi = P.RomInstance.load(path), O.Instance(path)
mu = g["mu"][k]
bbs = oi.boundary(*mu)
x, lam = g["x0"][k].copy(), g["lam0"][k].copy()
for it in range(nst):
    ev = O.eval_gradients(oi, bbs, x, lam)
    K = O.kkt_matrix(oi, ev)
    rhs = -ev.optimality
    s_o, l_o, reg = O.solve_kkt(oi, ev)
    sol = np.concatenate([s_o, l_o])
    res = np.linalg.norm(rhs - K @ sol) / np.linalg.norm(rhs)
    d = P.eval_gradients_batch(inst, mu[None], x[None], lam[None])
    nD = oi.n_primal
    dev = d.step[0]
    dres = np.linalg.norm(rhs - K @ dev) / np.linalg.norm(rhs)
    diag = np.abs(np.diag(K))
    print(f"it {it}: merit {ev.merit:.6e} dev {d.merit[0]:.6e}  oracle reg {reg} res {res:.2e} "
          f"dev status {d.kkt_status[0]} dev res(K) {dres:.2e} step rel "
          f"{np.abs(dev - sol).max() / np.abs(sol).max():.2e} |s| {np.abs(sol).max():.2e} "
          f"trace {np.trace(K[:nD, :nD]):.3e}")
    x = x + sol[:nD]
    lam = lam + sol[nD:]
