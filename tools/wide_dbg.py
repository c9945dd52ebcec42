import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DDNM_WIDE"] = "1"
import numpy as np
import paper_2305_15163_b200 as P
inst = P.RomInstance.load(os.path.join(ROOT, "tests", "golden", "c0_nm_artifacts.npz"))
for B in [int(a) for a in sys.argv[1:]]:
    mu = P.seeded_parameters(B, seed=1000)
    r = P.solve_rom_batch(inst, mu)
    print("B", B, "ok", r.seconds * 1e3, "ms", r.counters, flush=True)
