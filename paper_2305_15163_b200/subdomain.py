"""Subdomain sharding of the batched online solve.

In the reference every subdomain is one ``SqpBlock`` (sqp.py:28-41) whose
closures -- the HR residual chain of driver.py:404-432 and the constraint of
driver.py:366-378 -- are independent of the other blocks; ``eval_gradients``
(sqp.py:117-146) only sums their pieces and ``_kkt_matrix`` (sqp.py:149-159)
only places them.  So with many subdomains the blocks are split across ranks
(one process per GPU) and every SQP round of the whole mu batch is

1. ``eval``: this rank evaluates its contiguous block range at every running
   mu's trial point and packs, per mu, the block pieces the SQP needs (Gram
   block H_b = R_bᵀR_b, R_bᵀr_b, cval_b, cjac_b, r_bᵀr_b);
2. an all-gather of those packets (NCCL between GPUs, gloo in the CPU tests);
3. ``step``: the mu batch is split into contiguous slices, one per rank;
   each rank assembles, for the mu of its slice, all blocks' pieces in block
   order and runs the Armijo decision / KKT solve / trial update
   (sqp.py:230-299) -- every mu is solved by exactly one rank, so results
   are the one-rank results bit for bit and the KKT work (248 x 248 at
   config 4) divides by the rank count instead of being repeated;
4. an all-gather of the slices' trial records (running flag + the next trial
   point, n_D + 1 doubles per mu), which the next ``eval`` reads on every
   rank.  At the end the slices' results are all-gathered too.

Rounds are batch-synchronous: a mu that finished idles until the batch does.
The round engine is pluggable: :class:`DeviceRoundEngine` drives the
``ddnm_dd_*`` entry points of libddnm.so (include/ddnm.h); the CPU tests plug
an oracle-backed engine into the same host loop.
"""

from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

from . import _native as N
from .sqp import SqpConfig


def block_bounds(n_blocks: int, world: int) -> list:
    """Contiguous block ranges per rank: rank r owns [b[r], b[r+1]); sizes
    differ by at most one, lower ranks take the remainder."""
    if world < 1 or n_blocks < world:
        raise ValueError(f"cannot shard {n_blocks} blocks over {world} ranks")
    q, r = divmod(n_blocks, world)
    b = [0]
    for k in range(world):
        b.append(b[-1] + q + (1 if k < r else 0))
    return b


class DeviceRoundEngine:
    """Round engine on the GPU: k_dd_eval / k_dd_step through the C ABI.
    Packets live in torch CUDA tensors so torch.distributed (NCCL) can
    all-gather them on the current stream."""

    def __init__(self, instance, device: int = -1):
        import torch
        self.torch = torch
        self.inst = instance
        self.ctx = instance.context(device)
        self.dev = torch.device("cuda", self.ctx.info.device)
        self.h = None
        self.n_blocks = instance.n_blocks

    def packet_len(self, lo: int, hi: int) -> int:
        n = C.c_int64()
        N.check(N.lib().ddnm_dd_packet_len(self.ctx.h, lo, hi, C.byref(n)))
        return int(n.value)

    def buffer(self, n: int):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.dev)

    def _stream(self):
        return C.c_void_p(self.torch.cuda.current_stream(self.dev).cuda_stream)

    def begin(self, mu, cfg: SqpConfig, x0, lam0, lo: int, hi: int, rows: int = 0) -> int:
        """``rows`` >= B: output rows allocated (slices of equal size for the
        final all-gather); the device writes the first B."""
        from .driver import _cfg_struct
        t = self.torch
        B = mu.shape[0]
        R = max(rows, B)
        nD, nC, K = self.inst.n_primal, self.inst.n_mult, cfg.max_iter
        f64 = dict(dtype=t.float64, device=self.dev)
        i32 = dict(dtype=t.int32, device=self.dev)
        self.mu = t.as_tensor(mu, **f64).contiguous()
        self.x0 = None if x0 is None else t.as_tensor(np.asarray(x0, float).reshape(B, nD), **f64)
        self.lam0 = None if lam0 is None else t.as_tensor(np.asarray(lam0, float).reshape(B, nC), **f64)
        self.out = dict(
            x=t.zeros(R, nD, **f64), lam=t.zeros(R, nC, **f64), n_iter=t.zeros(R, **i32),
            n_evals=t.zeros(R, **i32), status=t.zeros(R, **i32), n_reg=t.zeros(R, **i32),
            merit=t.zeros(R, **f64), objective=t.zeros(R, **f64),
            merit_hist=t.zeros(R, K + 1, **f64), obj_hist=t.zeros(R, K + 1, **f64),
            alpha_hist=t.zeros(R, K, **f64), x0=t.zeros(R, nD, **f64), lam0=t.zeros(R, nC, **f64))
        self.B = B
        so = N.SolveOut()
        for k, v in self.out.items():
            ct = C.c_int32 if v.dtype == t.int32 else C.c_double
            setattr(so, k, C.cast(C.c_void_p(v.data_ptr()), C.POINTER(ct)))
        self.cfg = cfg
        h = C.c_void_p()
        n = C.c_int32()
        N.check(N.lib().ddnm_dd_begin(
            self.ctx.h, B, C.c_void_p(self.mu.data_ptr()),
            None if self.x0 is None else C.c_void_p(self.x0.data_ptr()),
            None if self.lam0 is None else C.c_void_p(self.lam0.data_ptr()),
            C.byref(_cfg_struct(cfg)), lo, hi, C.byref(so), self._stream(), C.byref(h),
            C.byref(n)))
        self.h = h
        return int(n.value)

    def trial_len(self) -> int:
        n = C.c_int64()
        N.check(N.lib().ddnm_dd_trial_len(self.h, C.byref(n)))
        return int(n.value)

    def set_trials(self, trials, mu_lo: int, mu_hi: int) -> None:
        """Trial records live in ``trials`` ([cap][trial_len], cap >= B);
        ``step`` then advances only mu in [mu_lo, mu_hi)."""
        cap = trials.numel() // self.trial_len()
        N.check(N.lib().ddnm_dd_set_trials(self.h, C.c_void_p(trials.data_ptr()), cap, mu_lo,
                                           mu_hi, self._stream()))

    def gather_results(self, rank: int, chunk: int, world: int, group) -> None:
        """Every rank's slice rows of every output to every rank."""
        for v in self.out.values():
            row = v.numel() // v.shape[0]
            flat = v.view(-1)
            _all_gather(flat, flat[rank * chunk * row:(rank + 1) * chunk * row].clone(), world,
                        group)

    def set_wide(self, on=True) -> None:
        """Evaluate with the batch-wide kernels (one lane per mu) instead of
        k_dd_eval.  ``True`` / 1: packets by lane with speculative step
        lengths (needs every block on this rank and ``wide_lanes`` packet
        rows); 2: one packet per mu as k_dd_eval writes them, for any block
        range (the ranks of a subdomain-sharded solve)."""
        N.check(N.lib().ddnm_dd_set_wide(self.h, int(on)))

    def eval(self, packets, stride: int) -> None:
        N.check(N.lib().ddnm_dd_eval(self.h, C.c_void_p(packets.data_ptr()), stride,
                                     self._stream()))

    def eval_p2p(self, peers, rank: int, stride: int) -> None:
        arr = (C.c_void_p * len(peers))(*[C.c_void_p(p) for p in peers])
        N.check(N.lib().ddnm_dd_eval_p2p(self.h, arr, len(peers), rank, stride, self._stream()))

    def step(self, gathered, nranks: int, bounds, stride: int, count: bool = True):
        """One round; returns the running-mu count, or None without a host
        synchronisation when ``count`` is False."""
        bnd = (C.c_int32 * len(bounds))(*bounds)
        n = C.c_int32()
        N.check(N.lib().ddnm_dd_step(self.h, C.c_void_p(gathered.data_ptr()), nranks, bnd,
                                     stride, self._stream(), C.byref(n) if count else None))
        return int(n.value) if count else None

    def finish(self, mu):
        from .driver import BatchResult
        self.torch.cuda.current_stream(self.dev).synchronize()
        out = {k: v[:self.B].cpu().numpy() for k, v in self.out.items()}
        N.lib().ddnm_dd_end(self.h)
        self.h = None
        return BatchResult(mu=mu, tol=self.cfg.tol, counters=self.ctx.counters(), **out)

    def __del__(self):
        h, self.h = getattr(self, "h", None), None
        if h:
            try:
                N.lib().ddnm_dd_end(h)
            except Exception:  # noqa: BLE001 -- interpreter shutdown
                pass


class ShardedSolve:
    """One rank's share of a subdomain-sharded batched solve.

    ``eval()`` returns this rank's packets ([B * stride] doubles); the caller
    all-gathers them rank-major into [world * B * stride] and passes that to
    ``step()``, which returns the number of mu still running."""

    def __init__(self, instance, mu, cfg: SqpConfig, rank: int, world: int, *, x0=None,
                 lam0=None, engine=None, device: int = -1, wide=None):
        self.eng = engine or DeviceRoundEngine(instance, device)
        nb = self.eng.n_blocks
        self.bounds = block_bounds(nb, world)
        self.rank, self.world = rank, world
        self.mu = mu
        self.B = mu.shape[0]
        self.stride = max(self.eng.packet_len(self.bounds[r], self.bounds[r + 1])
                          for r in range(world))
        self.lo, self.hi = self.bounds[rank], self.bounds[rank + 1]
        # mu slice of this rank's steps: equal slices (the all-gathers need
        # equal chunks), the last ones may run past B (empty records)
        self.chunk = -(-self.B // world)
        self.mu_lo = min(self.B, rank * self.chunk)
        self.mu_hi = min(self.B, (rank + 1) * self.chunk)
        self.active = self.eng.begin(mu, cfg, x0, lam0, self.lo, self.hi,
                                     rows=world * self.chunk)
        self.rec = self.eng.trial_len()
        self.trials = self.eng.buffer(world * self.chunk * self.rec)
        self.eng.set_trials(self.trials, self.mu_lo, self.mu_hi)
        self.packets = self.eng.buffer(self.B * self.stride)
        # this rank's blocks through the batch-wide kernels (one packet per mu,
        # same layout) when the instance has them: None = when eligible
        self.wide = False
        if isinstance(self.eng, DeviceRoundEngine) and wide is not False:
            if self.eng.ctx.info.wide:
                self.eng.set_wide(2)
                self.wide = True
            elif wide:
                raise NotImplementedError("instance not eligible for the wide evaluation")
        self.rounds = 0
        # every round evaluates one trial point per running mu; a solve takes
        # at most max_iter KKT steps of at most max_halvings + 1 trials each
        self.max_rounds = 2 + cfg.max_iter * (cfg.max_halvings + 1) + CHECK

    def eval(self):
        self.eng.eval(self.packets, self.stride)
        return self.packets

    def eval_p2p(self, peers):
        """Evaluation with the all-gather fused in: the kernel stores this
        rank's packets into every rank's gathered buffer (``peers[r]``, device
        addresses valid on this GPU) over peer memory."""
        self.eng.eval_p2p(peers, self.rank, self.stride)

    def step(self, gathered, count: bool = True):
        """One SQP round of this rank's mu slice: returns the slice's running
        count (``count=False``: None, no stream synchronisation; rounds after
        every mu finished do nothing, so a caller may check only every few
        rounds).  With several ranks the caller then all-gathers
        :meth:`trial_chunk` into :attr:`trials` and sums the counts."""
        n = self.eng.step(gathered, self.world, self.bounds, self.stride, count)
        self.rounds += 1
        if n is not None and n and self.rounds >= self.max_rounds:
            raise RuntimeError("sharded solve did not terminate within the SQP round bound")
        return n

    def trial_chunk(self):
        """This rank's slice of the trial records (its all-gather input)."""
        r = self.rank
        return self.trials[r * self.chunk * self.rec:(r + 1) * self.chunk * self.rec]

    def result(self, group=None):
        """The batch result; with several ranks every rank's slice rows are
        all-gathered first (collective over ``group``)."""
        if self.world > 1 and group is not False:
            self.eng.gather_results(self.rank, self.chunk, self.world, group)
        return self.eng.finish(self.mu)


CHECK = max(1, int(os.environ.get("DDNM_DD_CHECK", "4")))   # rounds between host reads of the running-mu count


def _all_gather(gathered, packets, world, group):
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(gathered, packets, group=group)
    else:
        dist.all_gather(list(gathered.view(world, -1).unbind(0)), packets, group=group)


class _DevBuffer:
    """A whole cudaMalloc allocation (CUDA IPC handles map allocations, not
    sub-allocations of torch's caching allocator)."""

    def __init__(self, nbytes: int, device: int):
        self.p = C.c_void_p()
        N.check(N.lib().ddnm_dev_alloc(device, nbytes, C.byref(self.p)))

    def data_ptr(self) -> int:
        return self.p.value

    def close(self):
        if self.p:
            N.lib().ddnm_dev_free(self.p)
            self.p = C.c_void_p()


class _PeerBuffers:
    """Every rank's gathered buffer mapped on this GPU (CUDA IPC handles
    exchanged over ``group``) for the fused peer-store all-gather."""

    def __init__(self, gathered, rank, world, group):
        import torch
        import torch.distributed as dist
        L = N.lib()
        h = C.create_string_buffer(64)
        err = None
        if L.ddnm_ipc_get_handle(C.c_void_p(gathered.data_ptr()), h) != 0:
            err = L.ddnm_last_error().decode(errors="replace")
        handles = [None] * world
        dist.all_gather_object(handles, None if err else h.raw, group=group)
        self.opened = []
        self.ptrs = []
        for r, hr in enumerate(handles):
            if r == rank:
                self.ptrs.append(gathered.data_ptr())
                continue
            if err or hr is None:
                err = err or f"rank {r} could not export its buffer"
                continue
            p = C.c_void_p()
            if L.ddnm_ipc_open_handle(hr, C.byref(p)) != 0:
                err = L.ddnm_last_error().decode(errors="replace")
                continue
            self.opened.append(p)
            self.ptrs.append(p.value)
        # every rank learns whether all mappings succeeded, so a failure on
        # one rank never leaves the others waiting in the round loop
        ok = torch.tensor([0.0 if err else 1.0], dtype=torch.float64,
                          device=torch.device("cuda", torch.cuda.current_device()))
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if ok.item() < 1.0:
            self.close()
            raise RuntimeError(f"peer-memory mapping failed: {err or 'on another rank'}")

    def close(self):
        for p in self.opened:
            N.lib().ddnm_ipc_close_handle(p)
        self.opened = []


def solve_rom_batch_subdomain_sharded(instance, mus, cfg: SqpConfig = SqpConfig(), *,
                                      x0=None, lam0=None, group=None, device: int = -1,
                                      engine=None, transport: str = "nccl", wide=None):
    """Batched ``solve_rom`` (driver.py:554-597, compute_error=False) with the
    subdomain blocks sharded over the ranks of ``group`` (every rank passes
    the same ``mus``); every rank returns the same full ``BatchResult``.

    ``transport``: ``"nccl"`` -- evaluation kernel, then an NCCL all-gather of
    the packets; ``"p2p"`` -- the evaluation kernel stores its packets into
    every rank's gathered buffer over peer memory (CUDA IPC between the
    processes of one node) and a one-element all-reduce orders the ranks
    before the step (device engine only).

    ``wide``: each rank evaluates its blocks with the batch-wide kernels (one
    lane per mu, csrc/ddnm_wide.h; one packet per mu, the same exchange and
    steps).  ``None``: when the instance is eligible and the transport is
    ``"nccl"`` (the fused peer stores are k_dd_eval's); ``False``: k_dd_eval."""
    if transport not in ("nccl", "p2p"):
        raise ValueError("transport must be 'nccl' or 'p2p'")
    import torch.distributed as dist

    from .driver import _mu_array
    mu = _mu_array(mus)
    dist_on = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if dist_on else 0
    world = dist.get_world_size(group) if dist_on else 1
    t0 = time.perf_counter()
    if transport == "p2p":
        if wide:
            raise ValueError("the wide evaluation goes with transport='nccl'")
        wide = False
    sh = ShardedSolve(instance, mu, cfg, rank, world, x0=x0, lam0=lam0, engine=engine,
                      device=device, wide=wide)
    active = sh.active
    peers, own = [], []
    if transport == "p2p" and world > 1:
        # two whole allocations per rank (IPC maps allocations), alternating
        # by round: a peer's evaluation of round t + 1 may start while this
        # rank's step of round t still reads; the all-reduce of round t + 1
        # orders every step of round t before any store of round t + 2
        try:
            for _ in range(2):
                own.append(_DevBuffer(world * sh.B * sh.stride * 8, sh.eng.dev.index))
                peers.append(_PeerBuffers(own[-1], rank, world, group))
        except Exception:
            for pb in peers:
                pb.close()
            for b in own:
                b.close()
            raise
        bufs = own
        ptrs = [pb.ptrs for pb in peers]
    else:
        g1 = sh.packets if world == 1 else sh.eng.buffer(world * sh.B * sh.stride)
        bufs = [g1, g1]
        ptrs = [[g1.data_ptr()]] * 2
    flag = sh.eng.buffer(1) if transport == "p2p" and world > 1 else None
    cnt = sh.eng.buffer(1) if world > 1 else None
    done = False
    try:
        while active:
            gathered = bufs[sh.rounds % 2]
            if transport == "p2p":
                sh.eval_p2p(ptrs[sh.rounds % 2])
                if world > 1:
                    dist.all_reduce(flag, group=group)     # orders every rank's stores
            else:
                packets = sh.eval()
                if world > 1:
                    _all_gather(gathered, packets, world, group)
            # the running count is read (one host sync) every CHECK rounds;
            # rounds after the last mu finished are empty launches
            check = sh.rounds % CHECK == CHECK - 1
            n = sh.step(gathered, count=check)
            if world > 1:
                # every rank's next trial points (its slice) to every rank
                _all_gather(sh.trials, sh.trial_chunk().clone(), world, group)
                if check:
                    cnt.fill_(float(n))
                    dist.all_reduce(cnt, group=group)
                    n = int(cnt.item())
            if check:
                active = n
        done = True
    finally:
        if own:
            # no evaluation kernel may still store through a peer mapping
            sh.eng.torch.cuda.current_stream(sh.eng.dev).synchronize()
        for pb in peers:
            pb.close()
        if own and done:
            dist.barrier(group=group)   # every rank unmapped before the frees
            for b in own:
                b.close()
        # on the error path the exported buffers are leaked rather than freed:
        # a peer may still have them mapped
    res = sh.result(group)
    if hasattr(res, "seconds"):
        res.seconds = time.perf_counter() - t0
        res.rounds = sh.rounds
    return res
