"""Small end-to-end cases through every kernel family (for debug builds with
bounds checks, and under compute-sanitizer): the persistent solve and the
evaluation on tiny / c0 / variants / evaluation units (c3_nm, forced on
tiny_nm), a generated latent pair (tiny42_nm), the KG kernels (c0_lss, dd16: KKT
workspace in L2, 96-row block path), the subdomain round kernels (NCCL-style
and fused peer stores, several rank states), the decoder and a context from
a binio instance file."""
import ctypes as C
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_15163_b200 as P  # noqa: E402
from paper_2305_15163_b200 import _native as N  # noqa: E402
from paper_2305_15163_b200.subdomain import ShardedSolve  # noqa: E402


def load(name):
    return P.RomInstance.load(os.path.join(ROOT, "tests", "golden", f"{name}_artifacts.npz"))


os.environ["DDNM_UNIT_ROWS"] = "24"          # evaluation units (the configs-3/4 path) on tiny
unit_inst = load("tiny_nm")
unit_inst.context()
del os.environ["DDNM_UNIT_ROWS"]
r = P.solve_rom_batch(unit_inst, P.seeded_parameters(6, seed=4))
print("tiny_nm units ok", unit_inst.context().info.eval_units, r.n_iter.tolist(), flush=True)
for name in ("tiny_nm", "tiny_ls", "c0_nm", "tiny_srpc", "c0_nmg", "c0_lss", "dd16_nm", "tiny42_nm",
             "c3_nm"):
    inst = load(name)
    mu = P.seeded_parameters(6, seed=4)
    r = P.solve_rom_batch(inst, mu)
    ev = P.eval_gradients_batch(inst, mu[:3], r.x0[:3], r.lam0[:3])
    if inst.has_full_decoders:
        P.decode_batch(inst, r.x)
    print(name, "ok", r.n_iter.tolist(), float(ev.merit[0]), flush=True)

inst = load("dd16_nm")
mu = P.seeded_parameters(5, seed=9)
one = P.solve_rom_batch_subdomain_sharded(inst, mu, wide=False)     # k_dd_eval, like the peer-store path
p2p = P.solve_rom_batch_subdomain_sharded(inst, mu, transport="p2p")
assert np.array_equal(one.x, p2p.x)
wide = P.solve_rom_batch_subdomain_sharded(inst, mu)                 # the ranks' blocks by the wide kernels
assert np.array_equal(wide.x, P.solve_rom_batch(inst, mu, engine="wide").x)
cfg = P.SqpConfig(max_iter=3)
ranks = [ShardedSolve(inst, mu, cfg, r, 3, wide=False) for r in range(3)]
n = 3 * ranks[0].B * ranks[0].stride
bufs = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in ranks]
active = ranks[0].active
while active:
    for sh in ranks:
        sh.eval_p2p([b.data_ptr() for b in bufs])
    active = sum(sh.step(b) for sh, b in zip(ranks, bufs))   # each rank its mu slice
    chunks = [sh.trial_chunk().clone() for sh in ranks]      # the trial all-gather
    for sh in ranks:
        for r, c in enumerate(chunks):
            sh.trials[r * c.numel():(r + 1) * c.numel()] = c
print("dd16 sharded ok", one.n_iter.tolist(), flush=True)

with tempfile.TemporaryDirectory() as d:
    inst = load("c0_nm")
    inst.save_binio(os.path.join(d, "c0.bin"))
    h = C.c_void_p()
    N.check(N.lib().ddnm_ctx_create_binio(-1, os.path.join(d, "c0.bin").encode(), 0, C.byref(h)))
    N.lib().ddnm_ctx_destroy(h)
print("binio ctx ok", flush=True)
