"""Batch-wide evaluation vs the slot kernels on one instance:
1. packets of one round (wide vs k_dd_eval) at the initial trial points;
2. whole solves, persistent kernel vs DDNM_WIDE=1 (x, lambda, n_iter);
3. timings of both.
Usage: wide_check.py [instance] [B]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_15163_b200 as P  # noqa: E402
from paper_2305_15163_b200.subdomain import DeviceRoundEngine  # noqa: E402
from paper_2305_15163_b200.sqp import SqpConfig  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c0_nm"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
inst = P.RomInstance.load(os.path.join(ROOT, "tests", "golden", f"{name}_artifacts.npz"))
mu = P.seeded_parameters(B, seed=1000)
cfg = SqpConfig()
nb = inst.n_blocks

# 1. packets of the first round
pk = {}
for wide in (False, True):
    eng = DeviceRoundEngine(inst)
    eng.begin(mu, cfg, None, None, 0, nb)
    stride = eng.packet_len(0, nb)
    if wide:
        eng.set_wide(True)
    rows = max(2 * ((B + 31) // 32 * 32), 1024) if wide else B
    packets = eng.buffer(rows * stride)
    eng.eval(packets, stride)
    torch.cuda.synchronize()
    pk[wide] = packets.cpu().numpy().reshape(rows, stride)[:B]
    eng.finish(mu)
a, b = pk[False], pk[True]
scale = np.abs(a).max(axis=0, keepdims=True) + 1e-300
print(f"{name} B={B}: packets wide vs slots: max rel (per column scale) {np.max(np.abs(a - b) / scale):.3e}, "
      f"max abs {np.abs(a - b).max():.3e}, |a| max {np.abs(a).max():.3e}")

# 2./3. whole solves
os.environ["DDNM_WIDE"] = "0"
for _ in range(2):
    r0 = P.solve_rom_batch(inst, mu)
os.environ["DDNM_WIDE"] = "1"
for _ in range(3):
    r1 = P.solve_rom_batch(inst, mu)
dx = np.max(np.abs(r0.x - r1.x), axis=1) / np.max(np.abs(r0.x), axis=1)
dl = np.max(np.abs(r0.lam - r1.lam), axis=1) / np.maximum(np.max(np.abs(r0.lam), axis=1), 1e-300)
print(f"solves: slots {r0.seconds*1e3:.2f} ms, wide {r1.seconds*1e3:.2f} ms; "
      f"x rel {dx.max():.3e}, lam rel {dl.max():.3e}, n_iter equal {int((r0.n_iter == r1.n_iter).sum())}/{B}, "
      f"status equal {int((r0.status == r1.status).sum())}/{B}, evals {r0.counters} vs {r1.counters}")
