"""mu-batch sharding across GPUs (one process per GPU).

The online solves of different parameters are independent, so
the batch is split into contiguous shards with no collective on the data
path; an optional all-gather at the end reassembles the per-mu results in
the original order on every rank.  Backend-agnostic: NCCL between GPUs,
gloo in the CPU tests (tests/test_sharding.py).
"""

from __future__ import annotations

import numpy as np

from .sqp import SqpConfig


def shard_range(B: int, rank: int, world: int) -> tuple:
    """Contiguous [lo, hi) of rank ``rank``: sizes differ by at most one,
    lower ranks take the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank/world")
    if B < 0:
        raise ValueError("negative batch")
    q, r = divmod(B, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


_FIELDS = ("x", "lam", "n_iter", "n_evals", "status", "n_reg", "merit", "objective",
           "merit_hist", "obj_hist", "alpha_hist", "x0", "lam0")


def solve_rom_batch_sharded(instance, mus, cfg: SqpConfig = SqpConfig(), *, x0=None,
                            lam0=None, group=None, gather: bool = True, solve_fn=None,
                            device: int = -1):
    """Solve this rank's shard of ``mus`` and (optionally) all-gather.

    Returns ``(lo, hi, local_result, gathered)``; ``gathered`` maps each
    result field to the full (B, ...) array in the original mu order (None
    when ``gather`` is False).  ``solve_fn`` defaults to
    :func:`driver.solve_rom_batch` (the device path)."""
    import torch.distributed as dist

    from .driver import _mu_array, solve_rom_batch
    mu = _mu_array(mus)
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    lo, hi = shard_range(mu.shape[0], rank, world)
    fn = solve_fn or solve_rom_batch
    kw = {}
    if x0 is not None:
        kw["x0"] = np.asarray(x0)[lo:hi]
    if lam0 is not None:
        kw["lam0"] = np.asarray(lam0)[lo:hi]
    if fn is solve_rom_batch:
        kw["device"] = device
    res = fn(instance, mu[lo:hi], cfg, **kw)
    if not gather:
        return lo, hi, res, None
    local = {f: np.asarray(getattr(res, f)) for f in _FIELDS}
    if world == 1:
        return lo, hi, res, local
    parts = [None] * world
    dist.all_gather_object(parts, (lo, hi, local), group=group)
    parts.sort(key=lambda p: p[0])
    out = {f: np.concatenate([p[2][f] for p in parts], axis=0) for f in _FIELDS}
    return lo, hi, res, out
