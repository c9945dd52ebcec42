import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2305_15163_b200 as P
inst = P.RomInstance.load('/root/repo/tests/golden/c0_nm_artifacts.npz')
mu = P.seeded_parameters(4096, seed=1000)
r = P.solve_rom_batch(inst, mu)
ne = r.n_evals
print('n_evals percentiles', {p: int(np.percentile(ne, p)) for p in (50, 75, 90, 95, 99, 99.9, 100)})
print('status counts', np.bincount(r.status), 'n_iter max', r.n_iter.max(), 'mean', r.n_iter.mean())
srt = np.sort(ne)[::-1]
print('top 20 n_evals', srt[:20])
# active count per round
rounds = np.arange(1, ne.max() + 1)
act = [(ne >= k).sum() for k in rounds]
print('active at round', {int(k): int(act[k - 1]) for k in (1, 10, 15, 20, 25, 30, 40, 50, 60, 80, 100, 150, 188) if k <= ne.max()})
print('sum active', sum(act), 'rounds with <=32 active', sum(1 for a in act if a <= 32), 'rounds <=256', sum(1 for a in act if a <= 256))
ah = r.alpha_hist
print('accepted alpha < 1 fraction', np.nanmean((ah < 1.0)[~np.isnan(ah)]))
