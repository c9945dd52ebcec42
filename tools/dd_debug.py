"""Debug: a 2-rank in-process sharded solve vs the 1-rank solve."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2305_15163_b200 as P
from paper_2305_15163_b200.subdomain import ShardedSolve
name = sys.argv[1] if len(sys.argv) > 1 else "dd16_nm"
inst = P.RomInstance.load(f'tests/golden/{name}_artifacts.npz')
mu = P.seeded_parameters(4, seed=4)
cfg = P.SqpConfig()
one = ShardedSolve(inst, mu, cfg, 0, 1)
two = [ShardedSolve(inst, mu, cfg, r, 2) for r in range(2)]
b = two[0].bounds
lens = [two[0].eng.packet_len(b[r], b[r + 1]) for r in range(2)]
print(name, "bounds", b, "lens", lens, "stride1", one.stride, "stride2", two[0].stride)
for rnd in range(2):
    p1 = one.eval().clone().view(4, -1).cpu().numpy()
    p2 = [sh.eval().clone() for sh in two]
    q = [p.view(4, -1).cpu().numpy() for p in p2]
    d0 = np.abs(q[0][:, :lens[0]] - p1[:, :lens[0]]).max()
    d1 = np.abs(q[1][:, :lens[1]] - p1[:, lens[0]:lens[0] + lens[1]]).max()
    print("round", rnd, "rank0 diff", d0, "rank1 diff", d1, "nan", np.isnan(p1).sum(), np.isnan(q[0]).sum(), np.isnan(q[1]).sum())
    g = torch.cat(p2)
    gg = g.view(2, 4, -1).cpu().numpy()
    print("  gathered vs packets", np.abs(gg[0] - q[0]).max(), np.abs(gg[1] - q[1]).max())
    a1 = one.step(one.packets)
    a2 = [sh.step(g) for sh in two]
    torch.cuda.synchronize()
    print("  active", a1, a2)
    for nm, sh in (("one", one), ("r0", two[0]), ("r1", two[1])):
        o = sh.eng.out
        print("   ", nm, "status", o["status"].tolist(), "lam0", o["lam0"][0, :4].tolist(), "x0", o["x0"][0, :3].tolist(), "merit_hist0", o["merit_hist"][:, 0].tolist())
