import sys, numpy as np
sys.path.insert(0, '.')
import paper_2305_15163_b200 as P
def L(n): return P.RomInstance.load(f'tests/golden/{n}_artifacts.npz')
pre = [L(n) for n in ("c0_nm", "dd16_nm", "tiny_srpc")]
for inst in pre:
    mu = P.seeded_parameters(64, seed=3)
    P.solve_rom_batch(inst, mu); P.solve_rom_batch_subdomain_sharded(inst, mu)
inst = L("c0_nmg")
mu = P.seeded_parameters(64, seed=3)
runs = {"mk": [P.solve_rom_batch(inst, mu) for _ in range(4)],
        "dd": [P.solve_rom_batch_subdomain_sharded(inst, mu) for _ in range(4)]}
for k, rs in runs.items():
    for i, r in enumerate(rs):
        d = np.argwhere(r.x != rs[0].x)
        print(k, i, "diff vs run0:", d[:5].tolist(), "status", np.bincount(r.status, minlength=4).tolist())
d = np.argwhere(runs["mk"][0].x != runs["dd"][0].x)
print("mk vs dd:", d[:10].tolist())
for (m, j) in d[:3]:
    print(m, j, runs["mk"][0].x[m, j], runs["dd"][0].x[m, j], runs["mk"][0].n_iter[m], runs["dd"][0].n_iter[m], runs["mk"][0].status[m], runs["dd"][0].status[m])
