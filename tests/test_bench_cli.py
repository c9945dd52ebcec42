"""bench.py's CPU-side contract: the reference arm runs here and prints one
JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

from .conftest import ROOT


def test_reference_arm_prints_one_json_line():
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--ref-seconds", "0.5"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "solves/s" and d["value"] > 0
    for k in ("metric", "n_gpus", "steps", "warmup", "higher_is_better", "config", "cpu_baseline",
              "e2e"):
        assert k in d, k
    assert d["cpu_baseline"]["kind"] == "port" and d["e2e"]["h2d_bytes_per_step"] == 0


def test_parity_block_against_committed_goldens():
    """The bench line's parity block (device results of the timed batch vs
    oracle + reference goldens), fed here with the oracle's own values."""
    import numpy as np
    import torch
    sys.path.insert(0, ROOT)
    import bench
    z = dict(np.load(bench.PARITY_FILE))
    outs = {"x": torch.from_numpy(z["oracle_x"].copy()),
            "lam": torch.from_numpy(z["oracle_lam"].copy()),
            "n_iter": torch.from_numpy(z["oracle_n_iter"].astype(np.int32))}
    p = bench.bench_parity(outs, 0)
    assert p["sample"] == 256 and p["oracle"]["pass"] and p["reference"]["pass"]
    assert p["oracle"]["n_iter_equal"] == 256 and p["reference"]["max_rel_x"] < 1e-12
    assert bench.bench_parity(outs, 5) is None        # a shard not starting at mu 0


def test_gpus_n_self_launches_one_rank_per_process():
    """`bench.py --gpus 2` without a torchrun environment launches the ranks
    itself (torch.distributed.run, 127.0.0.1); with the reference arm only
    rank 0 works and prints the single JSON line."""
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-seconds", "0.5"],
                         capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["scaling"] == "strong"
