"""Subdomain sharding: blocks split over ranks, per-round
all-gather of block pieces, identical SQP on every rank.

CPU tests run the shipping host loop (paper_2305_15163_b200/subdomain.py)
over gloo with world size 2 and 4, plugging in an oracle-backed round engine
(test infrastructure: packets hold the oracle's block pieces, the step drives
a generator restatement of oracle.solve).  GPU tests run the device engine
(k_dd_eval / k_dd_step) and compare it with the persistent megakernel, the
oracle and the reference goldens."""

import os
import socket

import numpy as np
import pytest

from oracle import ddnm_oracle as O

from .conftest import golden_path

DD = "dd16_nm"      # 60x60, 4x4 subdomains, n = (8, 5), n_C = 40 (config 4's layout)


def test_block_bounds():
    from paper_2305_15163_b200 import block_bounds
    assert block_bounds(16, 1) == [0, 16]
    assert block_bounds(16, 8) == list(range(0, 17, 2))
    assert block_bounds(4, 3) == [0, 2, 3, 4]
    for nb in (1, 4, 16):
        for w in range(1, nb + 1):
            b = block_bounds(nb, w)
            assert b[0] == 0 and b[-1] == nb and len(b) == w + 1
            sz = np.diff(b)
            assert sz.min() >= 1 and sz.max() - sz.min() <= 1
    with pytest.raises(ValueError):
        block_bounds(4, 5)
    with pytest.raises(ValueError):
        block_bounds(4, 0)


# -- oracle-backed round engine (CPU stand-in for DeviceRoundEngine) ----------

def _assemble(inst, pieces, lam):
    """oracle.eval_gradients (sqp.py:117-146) from per-block pieces."""
    rho = np.zeros(inst.n_primal)
    con = np.zeros(inst.n_c)
    evals = []
    for blk, off, (Br, R_int, R_gam, cval, cjac) in zip(inst.blocks, inst.offsets, pieces):
        rho[off:off + blk.n_int] = R_int.T @ Br
        rho[off + blk.n_int:off + blk.n_int + blk.n_gam] = R_gam.T @ Br + cjac.T @ lam
        con += cval
        evals.append((Br, R_int, R_gam, cval, cjac))
    return O.Eval(rho=rho, con=con, blocks=evals)


def _solve_gen(inst, a, lm, cfg):
    """oracle.solve (driver.py:554-597 + sqp.py:230-299) as a generator: it
    yields every point it needs evaluated and receives that point's block
    pieces (which do not depend on the multipliers)."""
    x0 = O.rbf_query(inst, a, lm)
    pieces = yield x0
    ev0 = _assemble(inst, pieces, np.zeros(inst.n_c))
    rows, rhs = [], []
    for off, blk, be in zip(inst.offsets, inst.blocks, ev0.blocks):
        gs = off + blk.n_int
        rows.append(be[4].T)
        rhs.append(-ev0.rho[gs:gs + blk.n_gam])
    lam0, *_ = np.linalg.lstsq(np.vstack(rows), np.concatenate(rhs), rcond=None)
    x = np.array(x0, dtype=float)
    lam = np.array(lam0, dtype=float)
    ev = _assemble(inst, pieces, lam)
    merits, alphas = [ev.merit], []
    best = (ev.merit, x.copy(), lam.copy())
    failure, n_iter, n_evals = None, 0, 1
    while merits[-1] >= cfg.tol and n_iter < cfg.max_iter:
        try:
            s, s_lam, _ = O.solve_kkt(inst, ev, cfg.reg_scale)
        except O.OracleConvergenceError:
            return x, lam, n_iter, n_evals, 2, merits
        alpha = 1.0
        accepted = None
        for _ in range(cfg.max_halvings + 1):
            pieces = yield x + alpha * s
            trial = _assemble(inst, pieces, lam + alpha * s_lam)
            n_evals += 1
            if trial.merit <= (1.0 - cfg.armijo_c1 * alpha) * merits[-1]:
                accepted = trial
                break
            alpha *= cfg.backtrack_factor
        if accepted is None:
            failure = "line_search"
            break
        x += alpha * s
        lam += alpha * s_lam
        ev = accepted
        n_iter += 1
        merits.append(ev.merit)
        alphas.append(alpha)
        if ev.merit < best[0]:
            best = (ev.merit, x.copy(), lam.copy())
    if failure is not None:
        _, x, lam = best
    return x, lam, n_iter, n_evals, 0 if failure is None else 1, merits


class OracleRoundEngine:
    """CPU stand-in for DeviceRoundEngine with the same protocol: trial
    records [running flag, x_trial] per mu, steps for a mu slice only,
    slice results gathered at the end."""

    def __init__(self, inst):
        self.inst = inst
        self.n_blocks = len(inst.blocks)
        self.nout = [b.weights.shape[0] if b.weights is not None else b.stencil.rows.size
                     for b in inst.blocks]
        self.plen = [r * (1 + b.n_int + b.n_gam) + inst.n_c * (1 + b.n_gam)
                     for r, b in zip(self.nout, inst.blocks)]
        self.evals = 0

    def packet_len(self, lo, hi):
        return sum(self.plen[lo:hi])

    def buffer(self, n):
        import torch
        return torch.zeros(n, dtype=torch.float64)

    def trial_len(self):
        return 1 + self.inst.n_primal

    def begin(self, mu, cfg, x0, lam0, lo, hi, rows=0):
        import torch
        assert x0 is None and lam0 is None
        self.lo, self.hi = lo, hi
        self.B = mu.shape[0]
        self.bbs = [self.inst.boundary(a, lm) for a, lm in mu]
        self.gens = [_solve_gen(self.inst, a, lm, cfg) for a, lm in mu]
        rec = self.trial_len()
        self.trials = torch.zeros(self.B * rec, dtype=torch.float64)
        t = self.trials.numpy().reshape(self.B, rec)
        for k, g in enumerate(self.gens):
            t[k, 0], t[k, 1:] = 1.0, next(g)
        self.res = [None] * self.B
        self.mlo, self.mhi = 0, self.B
        return self.B

    def set_trials(self, trials, mu_lo, mu_hi):
        trials[:self.trials.numel()] = self.trials
        self.trials, self.mlo, self.mhi = trials, mu_lo, mu_hi

    def eval(self, packets, stride):
        pk = packets.numpy()
        t = self.trials.numpy().reshape(-1, self.trial_len())
        for k in range(self.B):
            if t[k, 0] == 0.0:
                continue
            parts = self.inst.split(t[k, 1:])
            pos = k * stride
            for b in range(self.lo, self.hi):
                blk = self.inst.blocks[b]
                Br, R_int, R_gam = blk.residual(*parts[b], self.bbs[k][b])
                cval, cjac = blk.constraint(parts[b][1])
                flat = np.concatenate([Br, R_int.ravel(), R_gam.ravel(), cval,
                                       np.atleast_2d(cjac).ravel()])
                assert flat.size == self.plen[b]
                pk[pos:pos + flat.size] = flat
                pos += flat.size
                self.evals += 1

    def _unpack(self, flat, b):
        blk, nc = self.inst.blocks[b], self.inst.n_c
        r, ni, ng = self.nout[b], blk.n_int, blk.n_gam
        sizes = [r, r * ni, r * ng, nc, nc * ng]
        Br, Ri, Rg, cv, cj = np.split(flat[:self.plen[b]], np.cumsum(sizes)[:-1])
        return Br, Ri.reshape(r, ni), Rg.reshape(r, ng), cv, cj.reshape(nc, ng)

    def step(self, gathered, nranks, bounds, stride, count=True):
        g = gathered.numpy().reshape(nranks, self.B, stride)
        t = self.trials.numpy().reshape(-1, self.trial_len())
        active = 0
        for k in range(self.mlo, self.mhi):
            if self.res[k] is not None:
                continue
            pieces = []
            for r in range(nranks):
                pos = 0
                for b in range(bounds[r], bounds[r + 1]):
                    pieces.append(self._unpack(g[r, k, pos:], b))
                    pos += self.plen[b]
            try:
                t[k, 1:] = self.gens[k].send(pieces)
                active += 1
            except StopIteration as stop:
                self.res[k] = stop.value
                t[k, 0] = 0.0
        return active if count else None

    def gather_results(self, rank, chunk, world, group):
        import torch.distributed as dist
        parts = [None] * world
        dist.all_gather_object(parts, self.res[self.mlo:self.mhi], group=group)
        self.res = [r for p in parts for r in p]

    def finish(self, mu):
        return self.res


def _worker(rank, world, port, out_dir, name, B):
    import torch.distributed as dist

    from paper_2305_15163_b200 import SqpConfig, seeded_parameters
    from paper_2305_15163_b200.subdomain import solve_rom_batch_subdomain_sharded
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    inst = O.Instance(golden_path(name, "artifacts"))
    eng = OracleRoundEngine(inst)
    res = solve_rom_batch_subdomain_sharded(inst, seeded_parameters(B, seed=5), SqpConfig(),
                                            engine=eng)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
             x=np.stack([r[0] for r in res]), lam=np.stack([r[1] for r in res]),
             n_iter=np.array([r[2] for r in res]), n_evals=np.array([r[3] for r in res]),
             status=np.array([r[4] for r in res]), block_evals=eng.evals)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,world,B", [("tiny_nm", 2, 4), (DD, 2, 2), (DD, 4, 2)])
def test_sharded_rounds_match_unsharded_oracle(tmp_path, name, world, B):
    """world ranks over gloo, each evaluating only its blocks: every rank ends
    with the same results, bitwise equal to the unsharded oracle solve, and
    the block evaluations split across the ranks."""
    import torch.multiprocessing as mp

    from paper_2305_15163_b200 import SqpConfig, block_bounds, seeded_parameters
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), name, B), nprocs=world,
             join=True)
    rs = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    for r in rs[1:]:
        for k in ("x", "lam", "n_iter", "n_evals", "status"):
            np.testing.assert_array_equal(r[k], rs[0][k])
    inst = O.Instance(golden_path(name, "artifacts"))
    mu = seeded_parameters(B, seed=5)
    total_evals = 0
    for k in range(B):
        ref = O.solve(inst, mu[k, 0], mu[k, 1], O.SqpConfig())
        np.testing.assert_array_equal(rs[0]["x"][k], ref.x)
        np.testing.assert_array_equal(rs[0]["lam"][k], ref.lam)
        assert rs[0]["n_iter"][k] == ref.n_iter
        assert rs[0]["n_evals"][k] == ref.n_evals
        total_evals += ref.n_evals
    bnd = block_bounds(len(inst.blocks), world)
    for r in range(world):
        assert rs[r]["block_evals"] == total_evals * (bnd[r + 1] - bnd[r])


# -- device engine -----------------------------------------------------------

def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c0_nm", DD, "tiny_srpc", "c0_nmg", "c0_ls", "c3s_nm",
                                  "c0_lss"])
def test_device_sharded_world1_equals_megakernel(name, gpu_instances):
    """One rank owning every block: the round kernels reproduce the
    persistent kernel bit for bit (same per-slot arithmetic)."""
    import paper_2305_15163_b200 as P
    inst = gpu_instances[name] if name in gpu_instances else P.RomInstance.load(
        golden_path(name, "artifacts"))
    mu = P.seeded_parameters(64, seed=3)
    ref = P.solve_rom_batch(inst, mu, engine="slots")   # the persistent kernel
    res = P.solve_rom_batch_subdomain_sharded(inst, mu, wide=False)   # k_dd_eval
    for k in ("x", "lam", "n_iter", "n_evals", "status", "n_reg", "merit", "objective",
              "x0", "lam0"):
        np.testing.assert_array_equal(getattr(res, k), getattr(ref, k), err_msg=k)
    np.testing.assert_array_equal(np.nan_to_num(res.merit_hist, nan=-1),
                                  np.nan_to_num(ref.merit_hist, nan=-1))


def _exchange_trials(ranks):
    """What the all-gather of the trial records does, for rank states in one
    process: every rank's slice into every rank's buffer."""
    chunks = [sh.trial_chunk().clone() for sh in ranks]
    for sh in ranks:
        for r, c in enumerate(chunks):
            n = c.numel()
            sh.trials[r * n:(r + 1) * n] = c


def _exchange_results(ranks):
    """The final all-gather of the slices' result rows, in one process."""
    for k in ranks[0].eng.out:
        rows = [sh.eng.out[k][sh.rank * sh.chunk:(sh.rank + 1) * sh.chunk].clone() for sh in ranks]
        for sh in ranks:
            for r, c in enumerate(rows):
                sh.eng.out[k][r * sh.chunk:(r + 1) * sh.chunk] = c


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 16])
def test_device_sharded_ranks_in_one_process(world):
    """world rank states on one GPU, run one after the other in one process
    (no rank waits on another): each evaluates only its block range, the
    packets are concatenated rank-major (what the all-gather produces), and
    every rank's result equals the one-rank solve bitwise."""
    import torch

    import paper_2305_15163_b200 as P
    from paper_2305_15163_b200.subdomain import ShardedSolve
    inst = P.RomInstance.load(golden_path(DD, "artifacts"))
    mu = P.seeded_parameters(24, seed=4)
    one = P.solve_rom_batch_subdomain_sharded(inst, mu)
    cfg = P.SqpConfig()
    ranks = [ShardedSolve(inst, mu, cfg, r, world) for r in range(world)]
    gathered = torch.empty(world * ranks[0].B * ranks[0].stride, dtype=torch.float64,
                           device="cuda")
    active = ranks[0].active
    while active:
        parts = [sh.eval().clone() for sh in ranks]
        torch.cat(parts, out=gathered)
        active = sum(sh.step(gathered) for sh in ranks)    # each rank steps its mu slice
        _exchange_trials(ranks)
    _exchange_results(ranks)
    for sh in ranks:
        r = sh.result(group=False)
        for k in ("x", "lam", "n_iter", "n_evals", "status", "merit"):
            np.testing.assert_array_equal(getattr(r, k), getattr(one, k), err_msg=k)


@pytest.mark.gpu
def test_device_sharded_matches_reference_goldens():
    """dd16 (16 subdomains, n_C = 40) against the reference's own solves."""
    import paper_2305_15163_b200 as P
    g = dict(np.load(golden_path(DD, "golden")))
    inst = P.RomInstance.load(golden_path(DD, "artifacts"))
    res = P.solve_rom_batch_subdomain_sharded(inst, g["mu"])
    for k in range(g["mu"].shape[0]):
        assert _rel(res.x[k], g["x"][k]) < 1e-9, k
        assert _rel(res.lam[k], g["lam"][k]) < 1e-9, k
        assert res.status[k] == g["failure"][k], k
    oi = O.Instance(golden_path(DD, "artifacts"))
    for k in range(g["mu"].shape[0]):
        r = O.solve(oi, *g["mu"][k])
        if min(r.margins) > 1e-13 * r.merit_history[0]:
            assert res.n_iter[k] == r.n_iter == g["n_iter"][k], k


@pytest.mark.gpu
@pytest.mark.parametrize("B", [1, 7])
def test_device_sharded_edge_cases(B):
    """Given x0 / lam0, a short max_iter, batches that do not fill a CTA:
    the round kernels still reproduce the persistent kernel bit for bit."""
    import paper_2305_15163_b200 as P
    inst = P.RomInstance.load(golden_path("c0_nm", "artifacts"))
    mu = P.seeded_parameters(B, seed=21)
    cfg = P.SqpConfig(max_iter=3)
    base = P.solve_rom_batch(inst, mu, cfg, engine="slots")
    x0 = base.x0 * (1.0 + 1e-3)
    for kw in ({}, {"x0": x0}, {"x0": x0, "lam0": base.lam0}):
        ref = P.solve_rom_batch(inst, mu, cfg, engine="slots", **kw)
        res = P.solve_rom_batch_subdomain_sharded(inst, mu, cfg, wide=False, **kw)
        for k in ("x", "lam", "n_iter", "n_evals", "status", "x0", "lam0"):
            np.testing.assert_array_equal(getattr(res, k), getattr(ref, k), err_msg=f"{k} {kw.keys()}")
        assert np.all(res.n_iter <= 3)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 4])
def test_device_fused_peer_gather(world):
    """The fused evaluation + all-gather (k_dd_eval storing every rank's slice
    straight into every rank's gathered buffer): world rank states in one
    process, one GPU, run one after another; results equal the one-rank
    solve bitwise on every rank."""
    import torch

    import paper_2305_15163_b200 as P
    from paper_2305_15163_b200.subdomain import ShardedSolve
    inst = P.RomInstance.load(golden_path(DD, "artifacts"))
    mu = P.seeded_parameters(20, seed=8)
    one = P.solve_rom_batch_subdomain_sharded(inst, mu, wide=False)
    if world == 1:
        res = P.solve_rom_batch_subdomain_sharded(inst, mu, transport="p2p")
        for k in ("x", "lam", "n_iter", "status"):
            np.testing.assert_array_equal(getattr(res, k), getattr(one, k), err_msg=k)
        return
    cfg = P.SqpConfig()
    ranks = [ShardedSolve(inst, mu, cfg, r, world, wide=False) for r in range(world)]
    n = world * ranks[0].B * ranks[0].stride
    gathered = [torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
                for _ in ranks]
    ptrs = [g.data_ptr() for g in gathered]
    active = ranks[0].active
    while active:
        for sh in ranks:
            sh.eval_p2p(ptrs)
        active = sum(sh.step(g) for sh, g in zip(ranks, gathered))
        _exchange_trials(ranks)
    _exchange_results(ranks)
    for sh in ranks:
        r = sh.result(group=False)
        for k in ("x", "lam", "n_iter", "n_evals", "status"):
            np.testing.assert_array_equal(getattr(r, k), getattr(one, k), err_msg=k)


@pytest.mark.gpu
def test_ipc_handle_of_a_device_buffer():
    """The exported gathered buffer is a whole allocation (a CUDA IPC handle
    maps the start of the allocation holding the pointer) and the fused
    exchange runs on it."""
    import ctypes as C

    import torch

    import paper_2305_15163_b200 as P
    from paper_2305_15163_b200 import _native as N
    from paper_2305_15163_b200.subdomain import ShardedSolve, _DevBuffer
    inst = P.RomInstance.load(golden_path(DD, "artifacts"))
    mu = P.seeded_parameters(7, seed=2)
    one = P.solve_rom_batch_subdomain_sharded(inst, mu, wide=False)
    sh = ShardedSolve(inst, mu, P.SqpConfig(), 0, 1, wide=False)
    buf = _DevBuffer(sh.B * sh.stride * 8, torch.cuda.current_device())
    h = C.create_string_buffer(64)
    N.check(N.lib().ddnm_ipc_get_handle(C.c_void_p(buf.data_ptr()), h))
    assert any(h.raw)
    active = sh.active
    while active:
        sh.eval_p2p([buf.data_ptr()])
        active = sh.step(buf)
    r = sh.result()
    buf.close()
    np.testing.assert_array_equal(r.x, one.x)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_device_p2p_host_loop_protocol(world):
    """The host loop of solve_rom_batch_subdomain_sharded(transport="p2p")
    with several rank states in one process: two gathered-buffer sets
    alternating by round parity, the running count read only every CHECK-th
    round (count=False otherwise, no host synchronisation), each rank
    stepping its mu slice, trial records exchanged every round: bitwise the
    one-rank solve on every rank."""
    import torch

    import paper_2305_15163_b200 as P
    from paper_2305_15163_b200.subdomain import CHECK, ShardedSolve
    inst = P.RomInstance.load(golden_path(DD, "artifacts"))
    mu = P.seeded_parameters(19, seed=6)
    one = P.solve_rom_batch_subdomain_sharded(inst, mu, wide=False)
    ranks = [ShardedSolve(inst, mu, P.SqpConfig(), r, world, wide=False) for r in range(world)]
    n = world * ranks[0].B * ranks[0].stride
    bufs = [[torch.full((n,), float("nan"), dtype=torch.float64, device="cuda") for _ in ranks]
            for _ in range(2)]
    ptrs = [[b.data_ptr() for b in bset] for bset in bufs]
    active, rounds = ranks[0].active, 0
    while active:
        k = rounds % 2
        for sh in ranks:
            sh.eval_p2p(ptrs[k])
        check = rounds % CHECK == CHECK - 1
        counts = [sh.step(bufs[k][r], count=check) for r, sh in enumerate(ranks)]
        _exchange_trials(ranks)
        if check:
            active = sum(counts)
        else:
            assert all(c is None for c in counts)
        rounds += 1
    _exchange_results(ranks)
    for sh in ranks:
        r = sh.result(group=False)
        for key in ("x", "lam", "n_iter", "n_evals", "status"):
            np.testing.assert_array_equal(getattr(r, key), getattr(one, key), err_msg=key)


@pytest.mark.gpu
def test_device_sharded_config4_units():
    """Config 4 (960^2, 16 blocks as evaluation units): the mu-sharded rounds
    at 1 and 2 rank states reproduce the persistent kernel bit for bit, and
    the reference goldens to 1e-9."""
    import torch

    import paper_2305_15163_b200 as P
    from paper_2305_15163_b200.subdomain import ShardedSolve
    inst = P.RomInstance.load(golden_path("c4_nm", "artifacts"))
    g = dict(np.load(golden_path("c4_nm", "golden")))
    mu = g["mu"][:3]
    ref = P.solve_rom_batch(inst, mu, engine="slots")
    res = P.solve_rom_batch_subdomain_sharded(inst, mu, wide=False)
    for k in ("x", "lam", "n_iter", "status"):
        np.testing.assert_array_equal(getattr(res, k), getattr(ref, k), err_msg=k)
    for k in range(3):
        assert _rel(res.x[k], g["x"][k]) < 1e-9 and _rel(res.lam[k], g["lam"][k]) < 1e-9
    ranks = [ShardedSolve(inst, mu, P.SqpConfig(), r, 2, wide=False) for r in range(2)]
    gathered = torch.empty(2 * ranks[0].B * ranks[0].stride, dtype=torch.float64, device="cuda")
    active = ranks[0].active
    while active:
        torch.cat([sh.eval().clone() for sh in ranks], out=gathered)
        active = sum(sh.step(gathered) for sh in ranks)
        _exchange_trials(ranks)
    _exchange_results(ranks)
    for sh in ranks:
        r = sh.result(group=False)
        np.testing.assert_array_equal(r.x, ref.x)
        np.testing.assert_array_equal(r.n_iter, ref.n_iter)
