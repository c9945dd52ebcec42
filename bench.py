"""Benchmark: batched DD NM-ROM-HR SQP solves/sec on B200 (BASELINE.json metric).

Workload (BASELINE configs[2]): the 60x60, 2x2-subdomain
NM-ROM WFPC instance with collocation HR (n = (6, 4), n_C = 8, 180 rows per
subdomain; artifacts trained by the reference, tests/golden/c0_nm_*), a
fixed batch of 4096 seeded mu (seed 1000), FP64.  One "step" = one complete
batched ``solve_rom`` (device RBF init + least-squares multipliers + SQP
loop) over the whole batch.  Multi-GPU (BASELINE config 2: "then with the
batch sharded across 2, 4 and 8 GPUs"): the 4096 mu are split into
contiguous shards, one per rank, no data-path collective -- strong scaling;
weak scaling (4096 mu per GPU) is reported beside it.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

``--gpus N`` without a torchrun environment launches N ranks itself
(torch.distributed.run, 127.0.0.1).  ``--impl reference`` times the CPU
implementation of the same path (the numpy oracle port,
oracle/ddnm_oracle.py, all host cores) on a bounded sample of the workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ARTIFACT = os.path.join(ROOT, "tests", "golden", "c0_nm_artifacts.npz")
# many-subdomain instance for the subdomain-sharded path (config 4's layout)
DD_ARTIFACT = os.path.join(ROOT, "tests", "golden", "dd16_nm_artifacts.npz")
DD_BATCH = 256
METRIC = "DD NM-ROM-HR SQP solves/sec (batched mu)"
WORKLOAD = ("config2: 60x60 2x2 NM-ROM WFPC collocation HR, n=(6,4), n_C=8, 180 rows/sub, "
            "band 8 shift 1, 4096 seeded mu (seed 1000)")
UNIT = "solves/s"
BATCH = 4096
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peaks.json")


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# -- algorithmic work ---------------------------------------

def fp64_peak():
    try:
        with open(FP64_PEAK_FILE) as f:
            d = json.load(f)
        return float(d["dfma_tflops"]), "measured (tools/microbench/fp64_peaks.cu, DFMA)"
    except Exception:
        return 36.6, "measured earlier on this pool (DFMA)"


# -- clocks -------------------------------------------------------------------

class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# -- CPU (oracle port) ------------------------------------------------------------

def _cpu_worker(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import ddnm_oracle as O
    path, mus = args
    inst = O.Instance(path)
    for a, lam in mus:
        O.solve(inst, a, lam)
    return len(mus)


def cpu_solves_per_sec(mu: np.ndarray, seconds: float = 15.0):
    """Time the oracle port of solve_rom on all host cores over a bounded
    sample of the workload's mu; returns (solves/s, cores, sample)."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    per_core = max(1, int(round(seconds * 4.0)))   # ~4 solves/s/core at config 0
    n = min(mu.shape[0], per_core * cores)
    chunks = [(ARTIFACT, mu[i::cores][:per_core].tolist()) for i in range(cores)]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_worker, [(ARTIFACT, mu[:1].tolist())] * cores)   # warm import
        t0 = time.perf_counter()
        done = sum(pool.map(_cpu_worker, chunks))
        dt = time.perf_counter() - t0
    return done / dt, cores, f"{done} of the workload's seeded mu ({n} requested), {dt:.1f}s"


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import paper_2305_15163_b200 as P
    mu = P.seeded_parameters(BATCH, seed=1000)
    vals = []
    cores = os.cpu_count() or 1
    sample = ""
    for i in range(args.warmup + args.steps):
        v, cores, sample = cpu_solves_per_sec(mu[(i * 97) % 1024:], seconds=args.ref_seconds)
        if i >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded mu, reference-trained artifacts)",
        "config": {"workload": WORKLOAD, "global_batch": BATCH},
        "run": {"sample_per_step": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# -- GPU ---------------------------------------------------------------------------

def run_gpu(args):
    import ctypes as C

    import torch

    import paper_2305_15163_b200 as P
    from paper_2305_15163_b200 import _native as N
    from paper_2305_15163_b200.driver import _cfg_struct

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    inst = P.RomInstance.load(ARTIFACT)
    ctx = inst.context(local, args.slots)
    info = ctx.info
    cfg = P.SqpConfig()
    # strong scaling: the fixed 4096-mu batch, contiguous shard per rank
    mu_all = P.seeded_parameters(BATCH, seed=1000)
    lo, hi = rank * BATCH // world, (rank + 1) * BATCH // world
    B = hi - lo
    mu_h = np.ascontiguousarray(mu_all[lo:hi])
    mu_d = torch.from_numpy(mu_h).to(dev)
    nD, nC = info.n_primal, info.n_mult
    outs = {
        "x": torch.empty((B, nD), dtype=torch.float64, device=dev),
        "lam": torch.empty((B, nC), dtype=torch.float64, device=dev),
        "n_iter": torch.empty(B, dtype=torch.int32, device=dev),
        "n_evals": torch.empty(B, dtype=torch.int32, device=dev),
        "status": torch.empty(B, dtype=torch.int32, device=dev),
        "merit": torch.empty(B, dtype=torch.float64, device=dev),
    }
    def so_for(o):
        so = N.SolveOut()
        so.x = C.cast(C.c_void_p(o["x"].data_ptr()), C.POINTER(C.c_double))
        so.lam = C.cast(C.c_void_p(o["lam"].data_ptr()), C.POINTER(C.c_double))
        so.n_iter = C.cast(C.c_void_p(o["n_iter"].data_ptr()), C.POINTER(C.c_int32))
        so.n_evals = C.cast(C.c_void_p(o["n_evals"].data_ptr()), C.POINTER(C.c_int32))
        so.status = C.cast(C.c_void_p(o["status"].data_ptr()), C.POINTER(C.c_int32))
        so.merit = C.cast(C.c_void_p(o["merit"].data_ptr()), C.POINTER(C.c_double))
        return so
    so = so_for(outs)
    cs = _cfg_struct(cfg)
    stream = torch.cuda.Stream(dev)          # explicit (non-default) stream: events see the kernel
    L = N.lib()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > L2

    def step():
        N.check(L.ddnm_solve_batch_device(ctx.h, B, C.c_void_p(mu_d.data_ptr()), None, None,
                                          C.byref(cs), C.byref(so),
                                          C.c_void_p(stream.cuda_stream)))

    torch.cuda.set_stream(stream)
    mu_d = mu_d.clone()                        # allocated on the bench stream
    torch.cuda.synchronize()
    # engine: "auto" = the library's default (the batch-wide kernels when the
    # instance is eligible: one lane per mu, rounds of evaluation + SQP-step
    # kernels; else the persistent slot kernel)
    ctx.set_engine(args.engine)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    times, evals, kkts, launches, rounds = [], 0, 0, 0, 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(float(len(times)))           # L2 flush between timed steps
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            ev, kk = ctx.counters()
            evals += ev
            kkts += kk
            rd, ln = ctx.rounds()
            rounds += rd
            launches += ln
    torch.cuda.synchronize()
    total_ms = float(np.sum(times))
    if dist:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    value = BATCH * args.steps / (total_ms / 1e3)

    # the persistent slot kernel on the same batch, beside the headline
    # (reported, not the headline, when the default engine is the wide one)
    slot_engine = None
    if rounds > 0:
        ctx.set_engine("slots")
        outs_keep = {k: v.clone() for k, v in outs.items()}
        step()
        st = []
        for _ in range(min(args.steps, 5)):
            flush.fill_(2.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            st.append(e0.elapsed_time(e1))
        sms = float(np.median(st))
        if dist:
            t = torch.tensor([sms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sms = float(t.item())
        same = int((outs["n_iter"] == outs_keep["n_iter"]).sum().item())
        slot_engine = {"kernel": "k_solve (persistent: one CTA slot per mu, one launch)",
                       "ms_per_step": sms, "value": BATCH / (sms / 1e3), "unit": UNIT,
                       "n_iter_equal_to_headline_engine": same, "of": B}
        for k, v in outs_keep.items():
            outs[k].copy_(v)
        ctx.set_engine(args.engine)
        torch.cuda.synchronize()

    # parity of the timed batch (last timed step) against CPU goldens of its
    # first mu (tests/golden/bench_c0_parity.npz: oracle and reference
    # solve_rom on the same seed-1000 parameters, tools/make_bench_golden.py)
    parity = None
    if rank == 0:
        try:
            parity = bench_parity(outs, lo)
        except Exception as exc:      # reported, never fatal for the headline line
            parity = {"error": f"{type(exc).__name__}: {exc}"}

    # weak scaling beside it: 4096 mu per GPU (seed 1000 + rank)
    weak = None
    if not args.no_weak:
        weak = weak_scaling(P, N, C, torch, dist, ctx, cs, so_for, dev, stream, flush, rank, world, args)

    # full decode of the batch's solutions (RomInstance.decode, driver.py:148-152):
    # reported beside the solve, not part of `value`
    dec = None
    if inst.has_full_decoders:
        Lst = C.c_int64()
        N.check(L.ddnm_ctx_state_len(ctx.h, C.byref(Lst)))
        st_d = torch.empty((B, Lst.value), dtype=torch.float64, device=dev)

        def dstep():
            N.check(L.ddnm_decode_batch_device(ctx.h, B, C.c_void_p(outs["x"].data_ptr()), None,
                                               C.c_void_p(st_d.data_ptr()), None,
                                               C.c_void_p(stream.cuda_stream)))
        for _ in range(3):
            dstep()
        dts = []
        for _ in range(5):
            flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dstep()
            e1.record(stream)
            e1.synchronize()
            dts.append(e0.elapsed_time(e1))
        dms = float(np.median(dts))
        dec = {"kernel": "k_decode", "ms_per_batch": dms, "states_per_s": B / (dms / 1e3),
               "state_len": Lst.value, "bytes_written_per_batch": B * Lst.value * 8,
               "share_of_solve": dms / ms_per_step}
        del st_d

    # per-mu outcome of the last timed step (config summary)
    n_iter = outs["n_iter"].cpu().numpy()
    status = outs["status"].cpu().numpy()

    # end-to-end through the public API with host buffers
    e2e_vals = []
    res = None
    for i in range(max(2, min(args.steps, 5))):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        res = P.solve_rom_batch(inst, mu_h, cfg, slots=args.slots, engine=args.engine)
        e2e_vals.append(time.perf_counter() - t0)
    e2e_t = float(np.mean(e2e_vals[1:])) if len(e2e_vals) > 1 else e2e_vals[0]
    if dist:
        t = torch.tensor([e2e_t], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    K1 = cfg.max_iter + 1
    d2h = B * (nD * 8 * 2 + nC * 8 * 2 + 4 * 4 + 8 * 2 + K1 * 8 * 2 + cfg.max_iter * 8)
    e2e = {"value": BATCH / e2e_t, "unit": UNIT, "h2d_bytes_per_step": BATCH * 2 * 8,
           "d2h_bytes_per_step": d2h * world}

    sub = None
    if not args.no_subdomain:
        try:
            sub = subdomain_bench(P, torch, dist, world, dev, stream, flush)
        except Exception as exc:      # reported, never fatal for the headline line
            sub = {"error": f"{type(exc).__name__}: {exc}"}

    others = None
    if not args.no_subdomain:
        try:
            others = other_configs_bench(P, N, C, _cfg_struct, torch, dist, dev, stream, flush)
        except Exception as exc:      # reported, never fatal for the headline line
            others = {"error": f"{type(exc).__name__}: {exc}"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    from paper_2305_15163_b200.workmodel import eval_flops
    fl = eval_flops(inst.arrays, inst.meta)
    evals_per_step = evals / args.steps / inst.n_blocks      # mu-evals (all blocks)
    kkts_per_step = kkts / args.steps
    flops_per_step = evals_per_step * fl["per_eval"] + kkts_per_step * fl["kkt"]
    peak, peak_src = fp64_peak()
    achieved = flops_per_step / (ms_per_step / 1e3) / 1e12
    wide = rounds > 0
    prof_file = "r2w_ncu_summary.json" if wide else "r2_ncu_summary.json"
    traffic, kern_prof = None, None
    try:
        with open(os.path.join(ROOT, "profiles", prof_file)) as f:
            pj = json.load(f)
        traffic = pj["traffic_bytes_per_launch"]   # ncu --set full capture of the dominant kernel
        kern_prof = pj.get("kernels")
    except Exception:
        pass
    if wide:
        kernel = ("round loop of the batch-wide engine: k_wide_dec (hidden ring + banded decoder "
                  "sweep, the dominant kernel), k_wide_rows (stencil, chain rule, Gram, constraint), "
                  "k_dd_step2 (Armijo / KKT), k_wide_compact, k_wide_pack")
        tsrc = (f"dram__bytes_read+write of one full-batch k_wide_dec launch, profiles/{prof_file} "
                "(the g / Jacobian rows of 4096 lanes written once)")
    else:
        kernel = "k_solve (persistent SQP megakernel)"
        tsrc = (f"dram__bytes_read+write per launch, profiles/{prof_file} (1.25 MB weights + one "
                "write-back of the 16.6 MB per-slot L2 Jacobian-row scratch)")
    # achieved / frac: ALL algorithmic flops of the step (every kernel's) over
    # the whole step's device time; `kernels` = each kernel's share of the
    # step's device time and its own FP64-pipe utilisation (ncu, profiles/)
    roof = {"bound": "fp64", "achieved": round(achieved, 3), "peak": peak, "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "traffic_source": tsrc,
            "kernel": kernel,
            "kernels": kern_prof,
            "peak_source": peak_src,
            "algorithmic_flops_per_step": flops_per_step,
            "exp_per_step": evals_per_step * fl["exp_per_eval"],
            "mu_evals_per_step": evals_per_step, "kkt_solves_per_step": kkts_per_step,
            "flops_per_mu_eval": fl["per_eval"], "flops_per_kkt": fl["kkt"]}
    cpu = None
    if world == 1 and not args.no_cpu:
        v, cores, sample = cpu_solves_per_sec(mu_h, seconds=args.ref_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded mu; artifacts trained by the reference on the 6x6 mu grid)",
        "config": {"workload": WORKLOAD, "global_batch": BATCH},
        "run": {"batch_per_gpu": B,
                   "parallelism": f"mu-shard x{world} (contiguous shards of the fixed batch)",
                   "l2": "flushed (256 MB write) between timed steps",
                   "engine": "wide (one lane per mu)" if wide else "slots (persistent kernel)",
                   "sqp_rounds_per_step": rounds / args.steps,
                   "slots_per_cta": info.slots_per_cta, "ctas": info.ctas,
                   "mean_n_iter": float(n_iter.mean()), "status_counts": np.bincount(status, minlength=4).tolist()},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "slot_engine": slot_engine,
        "clocks": clk.summary(),
        "parity": parity,
        "weak_scaling": weak,
        "decode": dec,
        "subdomain": sub,
        "other_configs": others,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


PARITY_FILE = os.path.join(ROOT, "tests", "golden", "bench_c0_parity.npz")


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def bench_parity(outs, lo):
    """Rank 0's shard starts at mu `lo` = 0: compare its first mu with the
    CPU goldens of the same seed-1000 parameters (north-star gate: x, lam to
    1e-9 relative; identical iteration counts)."""
    if not os.path.exists(PARITY_FILE) or lo != 0:
        return None
    z = dict(np.load(PARITY_FILE))
    n = min(int(z["oracle_x"].shape[0]), outs["x"].shape[0])
    x = outs["x"][:n].cpu().numpy()
    lam = outs["lam"][:n].cpu().numpy()
    it = outs["n_iter"][:n].cpu().numpy()
    out = {"sample": n, "of_batch": "first mu of the timed seed-1000 batch", "tol": 1e-9}
    for who in ("oracle", "reference"):
        if f"{who}_x" not in z:
            continue
        ex = max(_rel(x[k], z[f"{who}_x"][k]) for k in range(n))
        el = max(_rel(lam[k], z[f"{who}_lam"][k]) for k in range(n))
        eq = int(np.sum(it == z[f"{who}_n_iter"][:n]))
        out[who] = {"max_rel_x": ex, "max_rel_lam": el, "n_iter_equal": eq,
                    "pass": bool(ex <= 1e-9 and el <= 1e-9)}
    if "robust" in z:
        rb = z["robust"][:n].astype(bool)
        out["robust_mu"] = int(rb.sum())
        out["n_iter_equal_on_robust"] = int(np.sum((it == z["oracle_n_iter"][:n])[rb]))
    return out


def weak_scaling(P, N, C, torch, dist, ctx, cs, so_for, dev, stream, flush, rank, world, args):
    """4096 mu per GPU (seed 1000 + rank): the weak-scaling extra."""
    B = BATCH
    mu = torch.from_numpy(P.seeded_parameters(B, seed=1000 + rank)).to(dev)
    nD, nC = ctx.info.n_primal, ctx.info.n_mult
    o = {"x": torch.empty((B, nD), dtype=torch.float64, device=dev),
         "lam": torch.empty((B, nC), dtype=torch.float64, device=dev),
         "n_iter": torch.empty(B, dtype=torch.int32, device=dev),
         "n_evals": torch.empty(B, dtype=torch.int32, device=dev),
         "status": torch.empty(B, dtype=torch.int32, device=dev),
         "merit": torch.empty(B, dtype=torch.float64, device=dev)}
    so = so_for(o)

    def launch():
        N.check(N.lib().ddnm_solve_batch_device(ctx.h, B, C.c_void_p(mu.data_ptr()), None, None,
                                                C.byref(cs), C.byref(so),
                                                C.c_void_p(stream.cuda_stream)))
    launch()
    times = []
    for _ in range(3):
        flush.fill_(4.0)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"batch_per_gpu": B, "value": world * B / (ms / 1e3), "unit": UNIT, "ms_per_batch": ms,
            "scaling": "weak"}


# the other BASELINE configs (strong scaling: each config's fixed batch, sharded)
OTHER_CONFIGS = [
    ("config1_ls", "c0_ls", 4096, "config1: 60x60 2x2 LS-ROM WFPC collocation HR, n=(20,8), "
                                  "n_C=16, 180 rows/sub"),
    ("config3_layout_120", "c3s_nm", 1024, "config 3's layout at 120x120: 2x2 NM-ROM, "
                                           "n=(8,5), n_C=10, 2% collocation rows (144/sub)"),
    ("config4_layout_dd16", "dd16_nm", 256, "config 4's layout at 60x60: 4x4 NM-ROM, "
                                            "n=(8,5), n_C=40, 45 rows/sub (persistent kernel)"),
    ("config3", "c3_nm", 1024, "config3: 480x480 2x2 NM-ROM WFPC, n=(8,5), n_C=10, 2% collocation "
                               "rows (2304/sub), blocks as evaluation units"),
    ("config4", "c4_nm", 256, "config4: 960x960 4x4 NM-ROM WFPC, n=(8,5), n_C=40, 2% collocation "
                              "rows (2304/sub), blocks as evaluation units"),
]


def other_configs_bench(P, N, C, cfg_struct, torch, dist, dev, stream, flush, reps=3):
    """Device-timed solves/s of the other BASELINE configs (CUDA events on the
    launching stream, L2 flushed between launches, max over ranks)."""
    out = {}
    for key, name, B, desc in OTHER_CONFIGS:
        path = os.path.join(ROOT, "tests", "golden", f"{name}_artifacts.npz")
        if not os.path.exists(path):
            continue
        inst = P.RomInstance.load(path)
        ctx = inst.context(dev.index)
        rank = dist.get_rank() if dist else 0
        world = dist.get_world_size() if dist else 1
        Bt = B
        lo, hi = rank * Bt // world, (rank + 1) * Bt // world
        B = hi - lo
        mu = torch.from_numpy(np.ascontiguousarray(P.seeded_parameters(Bt, seed=3000)[lo:hi])).to(dev)
        nD, nC = inst.n_primal, inst.n_mult
        x = torch.empty((B, nD), dtype=torch.float64, device=dev)
        lam = torch.empty((B, nC), dtype=torch.float64, device=dev)
        st = torch.empty(B, dtype=torch.int32, device=dev)
        it = torch.empty(B, dtype=torch.int32, device=dev)
        so = N.SolveOut()
        so.x = C.cast(C.c_void_p(x.data_ptr()), C.POINTER(C.c_double))
        so.lam = C.cast(C.c_void_p(lam.data_ptr()), C.POINTER(C.c_double))
        so.status = C.cast(C.c_void_p(st.data_ptr()), C.POINTER(C.c_int32))
        so.n_iter = C.cast(C.c_void_p(it.data_ptr()), C.POINTER(C.c_int32))
        cs = cfg_struct(P.SqpConfig())

        def launch():
            N.check(N.lib().ddnm_solve_batch_device(ctx.h, B, C.c_void_p(mu.data_ptr()), None,
                                                    None, C.byref(cs), C.byref(so),
                                                    C.c_void_p(stream.cuda_stream)))
        def timed(engine):
            ctx.set_engine(engine)
            launch()
            times = []
            for _ in range(reps):
                flush.fill_(3.0)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                launch()
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            ms = float(np.median(times))
            if dist:
                t = torch.tensor([ms], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            return ms
        # the slot kernel beside the default engine when that is the wide one
        slots_ms = timed("slots") if ctx.info.wide else None
        ms = timed("auto")
        rounds, _ = ctx.rounds()
        from paper_2305_15163_b200.workmodel import eval_flops
        evals, _ = ctx.counters()            # block evaluations of the last launch
        fl = eval_flops(inst.arrays, inst.meta)
        peak, _ = fp64_peak()
        # evaluation flops only (the KKT count depends on which LU path runs)
        eval_tf = evals / inst.n_blocks * fl["per_eval"] / (ms / 1e3) / 1e12 / world
        if dist:
            ev_t = torch.tensor([float(evals)], device=dev, dtype=torch.float64)
            dist.all_reduce(ev_t)
            evals = int(ev_t.item())
        out[key] = {"workload": desc, "batch": Bt, "scaling": "strong", "batch_per_gpu": B,
                    "solves_per_s": Bt / (ms / 1e3),
                    "ms_per_batch": ms, "mean_n_iter": float(it.float().mean().item()),
                    "status_counts": torch.bincount(st.long(), minlength=4).tolist(),
                    "engine": "wide" if rounds > 0 else "slots", "sqp_rounds": rounds,
                    "slot_engine_ms_per_batch": slots_ms,
                    "slots_per_cta": ctx.info.slots_per_cta, "eval_units": ctx.info.eval_units,
                    "eval_tflops": round(eval_tf, 3), "eval_frac_of_fp64_peak": round(eval_tf / peak, 4)}
    return out


def subdomain_bench(P, torch, dist, world, dev, stream, flush, reps=3):
    """dd16 (config 4's layout at 60x60) and, when its artifacts exist, config 4
    itself (960x960, 4x4, 256 mu) through the subdomain-sharded rounds."""
    out = {"dd16": _subdomain_one(P, torch, dist, world, dev, stream, flush, DD_ARTIFACT,
                                  DD_BATCH, "dd16: 60x60 4x4 NM-ROM WFPC collocation HR, "
                                  "n=(8,5), n_C=40, 45 rows/sub (config 4's layout at a "
                                  "trainable grid)", reps)}
    c4 = os.path.join(ROOT, "tests", "golden", "c4_nm_artifacts.npz")
    if os.path.exists(c4):
        out["config4"] = _subdomain_one(P, torch, dist, world, dev, stream, flush, c4, 256,
                                        "config4: 960x960 4x4 NM-ROM WFPC, n=(8,5), n_C=40, "
                                        "2304 rows/sub, blocks as evaluation units", 2,
                                        transports=("nccl",))
    return out


def _subdomain_one(P, torch, dist, world, dev, stream, flush, path, batch, desc, reps,
                   transports=("nccl", "p2p")):
    """The subdomain-sharded path: blocks sharded over the
    ranks with an exchange of the block packets every SQP round -- an NCCL
    all-gather after the evaluation kernel, or the evaluation kernel storing
    the packets into every rank's buffer over peer memory ("p2p", CUDA IPC)
    -- the steps sharded by mu (each mu's KKT on one rank, trial points
    all-gathered), strong scaling (the same batch at every N).  Device-timed
    with CUDA events, max over ranks."""
    inst = P.RomInstance.load(path)
    mu = P.seeded_parameters(batch, seed=2000)
    out = {"workload": desc, "batch": batch, "scaling": "strong", "ranks": world,
           "kernels": "per SQP round: each rank's blocks by the wide kernels (k_wide_dec / k_wide_rows, "
                      "one packet per mu) or by k_dd_eval (the *_slots entries and p2p), exchange, "
                      "k_dd_step on the rank's mu slice"}
    variants = []
    for transport in transports:
        if transport == "nccl":
            variants += [("nccl", "nccl", None), ("nccl_slots", "nccl", False)]
        else:
            variants.append((transport, transport, False))
    for key, transport, wide in variants:
        try:
            P.solve_rom_batch_subdomain_sharded(inst, mu, transport=transport, wide=wide)   # warm-up
            times, res = [], None
            for _ in range(reps):
                flush.fill_(2.0)
                if dist:
                    dist.barrier()
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                res = P.solve_rom_batch_subdomain_sharded(inst, mu, transport=transport, wide=wide)
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            ms = float(np.median(times))
            if dist:
                t = torch.tensor([ms], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            out[key] = {"solves_per_s": batch / (ms / 1e3), "ms_per_batch": ms,
                              "rounds": int(res.rounds), "mean_n_iter": float(res.n_iter.mean()),
                              "status_counts": np.bincount(res.status, minlength=4).tolist()}
        except Exception as exc:      # reported per transport, never fatal
            out[key] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-subdomain", action="store_true",
                    help="skip the extra measurements (subdomain-sharded dd16, other configs)")
    ap.add_argument("--slots", type=int, default=0, help="mu slots per CTA (0 = largest that fits)")
    ap.add_argument("--no-weak", action="store_true", help="skip the weak-scaling extra")
    ap.add_argument("--engine", default="auto", choices=["auto", "slots", "wide"],
                    help="solve engine of the headline (auto: the library's default)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: launch the ranks ourselves (the driver may also
        # launch us under torchrun, then WORLD_SIZE is set)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")            # init lines (ranks, transports) ...
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # ... on stderr, not in the JSON stream
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd, env=env)
    if "WORLD_SIZE" in os.environ:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
