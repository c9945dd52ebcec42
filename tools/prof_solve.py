"""One warm batched solve for profiling (ncu -k regex:k_solve -s 1 -c 1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2305_15163_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c0_nm"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
slots = int(sys.argv[3]) if len(sys.argv) > 3 else 0
inst = P.RomInstance.load(os.path.join(ROOT, "tests", "golden", f"{name}_artifacts.npz"))
mu = P.seeded_parameters(B, seed=1000)
for _ in range(3):
    r = P.solve_rom_batch(inst, mu, slots=slots)
ctx = inst.context(-1, slots)
print(f"slots/CTA {ctx.info.slots_per_cta}, CTAs {ctx.info.ctas}, smem {ctx.info.smem_bytes} B, "
      f"units {ctx.info.eval_units}")
prof = ctx.profile()
tot = sum(prof.values()) or 1
print({k: f"{100 * v / tot:.1f}%" for k, v in prof.items()})
print(f"{name} B={B} solve {r.seconds*1e3:.2f} ms, evals {r.counters}, mean n_iter {r.n_iter.mean():.2f}")
