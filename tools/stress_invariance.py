"""Stress: for every instance, per-mu results are bitwise independent of the
batch order, of repetition and of the path (persistent kernel vs
subdomain-sharded rounds)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2305_15163_b200 as P

names = ["tiny_nm", "tiny_ls", "c0_nm", "c0_ls", "c3s_nm", "tiny_nmg", "tiny_srpc", "tiny_lsg",
         "tiny_lss", "c0_nmg", "c0_srpc", "c0_lsg", "c0_lss", "dd16_nm"]
bad = []
for n in names:
    inst = P.RomInstance.load(f'tests/golden/{n}_artifacts.npz')
    mu = P.seeded_parameters(96, seed=77)
    perm = np.random.default_rng(5).permutation(mu.shape[0])
    a = P.solve_rom_batch(inst, mu)
    b = P.solve_rom_batch(inst, mu[perm])
    c = P.solve_rom_batch_subdomain_sharded(inst, mu)
    ok1 = np.array_equal(a.x[perm], b.x) and np.array_equal(a.n_iter[perm], b.n_iter)
    ok2 = np.array_equal(a.x, c.x) and np.array_equal(a.n_iter, c.n_iter)
    print(f"{n:10s} permutation {'ok' if ok1 else 'DIFF'}  sharded {'ok' if ok2 else 'DIFF'}", flush=True)
    if not (ok1 and ok2):
        bad.append(n)
print("bad:", bad)
