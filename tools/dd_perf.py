import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2305_15163_b200 as P
inst = P.RomInstance.load('tests/golden/dd16_nm_artifacts.npz')
for B in (256, 1024):
    mu = P.seeded_parameters(B, seed=9)
    for rep in range(2):
        torch.cuda.synchronize(); t=time.perf_counter()
        r1 = P.solve_rom_batch(inst, mu); t1=time.perf_counter()-t
        torch.cuda.synchronize(); t=time.perf_counter()
        r2 = P.solve_rom_batch_subdomain_sharded(inst, mu); t2=time.perf_counter()-t
    print(f"B={B} megakernel {t1*1e3:.1f} ms ({B/t1:.0f}/s)  round-sync {t2*1e3:.1f} ms ({B/t2:.0f}/s) same={np.array_equal(r1.x, r2.x)} iters={r1.n_iter.mean():.2f} status={np.bincount(r1.status, minlength=4)}")
print(inst.context().info.slots_per_cta, inst.context().info.ctas, inst.context().info.smem_bytes)
