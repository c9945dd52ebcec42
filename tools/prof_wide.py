"""Warm batched solves through the batch-wide path (for ncu launch lists)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("DDNM_WIDE", "1")
import paper_2305_15163_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c0_nm"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
inst = P.RomInstance.load(os.path.join(ROOT, "tests", "golden", f"{name}_artifacts.npz"))
mu = P.seeded_parameters(B, seed=1000)
for _ in range(reps):
    r = P.solve_rom_batch(inst, mu)
ctx = inst.context()
print(f"{name} B={B} wide={os.environ['DDNM_WIDE']} solve {r.seconds*1e3:.2f} ms, evals {r.counters}, "
      f"mean n_iter {r.n_iter.mean():.2f}, rounds {r.rounds}, lanes launched {ctx.lanes()} vs consumed "
      f"{int(r.n_evals.sum())}")
