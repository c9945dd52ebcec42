"""Multi-process (world size 2, gloo, CPU) tests of the mu-batch sharding.

The device solve is replaced by an injected CPU solver (the oracle) so the
sharding/gather logic runs here without a GPU; the product path itself is
covered by the -m gpu tests."""

import os
import socket

import numpy as np
import pytest

from paper_2305_15163_b200.sharding import shard_range


@pytest.mark.parametrize("B,world", [(0, 2), (1, 2), (7, 2), (4096, 8), (5, 3), (16, 1)])
def test_shard_range_partitions_batch(B, world):
    ranges = [shard_range(B, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == B
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1


def test_shard_range_rejects_bad_args():
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
    with pytest.raises(ValueError):
        shard_range(-1, 0, 1)


class _OracleBatch:
    """Mimics BatchResult fields from oracle solves (CPU stand-in)."""

    def __init__(self, inst, mu, cfg):
        from oracle import ddnm_oracle as O
        B = mu.shape[0]
        nD, nC, K = inst.n_primal, inst.n_c, cfg.max_iter
        self.x = np.zeros((B, nD)); self.lam = np.zeros((B, nC))
        self.n_iter = np.zeros(B, np.int32); self.n_evals = np.zeros(B, np.int32)
        self.status = np.zeros(B, np.int32); self.n_reg = np.zeros(B, np.int32)
        self.merit = np.zeros(B); self.objective = np.zeros(B)
        self.merit_hist = np.full((B, K + 1), np.nan); self.obj_hist = np.full((B, K + 1), np.nan)
        self.alpha_hist = np.full((B, K), np.nan)
        self.x0 = np.zeros((B, nD)); self.lam0 = np.zeros((B, nC))
        for k in range(B):
            r = O.solve(inst, mu[k, 0], mu[k, 1], O.SqpConfig(max_iter=cfg.max_iter))
            self.x[k], self.lam[k], self.n_iter[k] = r.x, r.lam, r.n_iter
            self.n_evals[k] = r.n_evals
            self.status[k] = 0 if r.failure_reason is None else 1
            self.merit[k], self.objective[k] = r.merit_history[-1], r.objective_history[-1]
            self.merit_hist[k, :len(r.merit_history)] = r.merit_history


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from oracle import ddnm_oracle as O
    from paper_2305_15163_b200 import SqpConfig, seeded_parameters
    from paper_2305_15163_b200.sharding import solve_rom_batch_sharded
    from tests.conftest import golden_path
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    inst = O.Instance(golden_path("tiny_nm", "artifacts"))
    mu = seeded_parameters(5, seed=11)
    cfg = SqpConfig(max_iter=4)
    lo, hi, local, full = solve_rom_batch_sharded(
        inst, mu, cfg, solve_fn=lambda i, m, c, **kw: _OracleBatch(i, m, c))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), lo=lo, hi=hi, **full)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_solve_gathers_in_order(tmp_path):
    import torch.multiprocessing as mp

    from oracle import ddnm_oracle as O
    from paper_2305_15163_b200 import SqpConfig, seeded_parameters
    from tests.conftest import golden_path
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r0 = dict(np.load(tmp_path / "rank0.npz"))
    r1 = dict(np.load(tmp_path / "rank1.npz"))
    assert (int(r0["lo"]), int(r0["hi"]), int(r1["lo"]), int(r1["hi"])) == (0, 3, 3, 5)
    for k in r0:
        if k not in ("lo", "hi"):
            np.testing.assert_array_equal(r0[k], r1[k])       # every rank has the full batch
    # and it equals the single-process answer, in the original order
    inst = O.Instance(golden_path("tiny_nm", "artifacts"))
    ref = _OracleBatch(inst, seeded_parameters(5, seed=11), SqpConfig(max_iter=4))
    np.testing.assert_array_equal(r0["x"], ref.x)
    np.testing.assert_array_equal(r0["n_iter"], ref.n_iter)
