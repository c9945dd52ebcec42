"""Small end-to-end case for compute-sanitizer (solve + eval on tiny and c0)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2305_15163_b200 as P  # noqa: E402

for name in ("tiny_nm", "tiny_ls", "c0_nm"):
    inst = P.RomInstance.load(os.path.join(ROOT, "tests", "golden", f"{name}_artifacts.npz"))
    mu = P.seeded_parameters(24, seed=4)
    r = P.solve_rom_batch(inst, mu)
    ev = P.eval_gradients_batch(inst, mu[:5], r.x0[:5], r.lam0[:5])
    print(name, "ok", r.n_iter[:6].tolist(), float(ev.merit[0]))
