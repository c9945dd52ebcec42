"""profiles/r2w_ncu_summary.json from the round's ncu captures:
  launches.csv   ncu --metrics gpu__time_duration.sum launch list of bench.py (one timed step)
  dec/rows/step  ncu --set full captures (.ncu-rep) of one full-batch launch of each kernel
usage: ncu_summary_wide.py launches.csv dec.ncu-rep rows.ncu-rep step.ncu-rep out.json"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

launches, reps, out = sys.argv[1], sys.argv[2:5], sys.argv[5]
WANT = {
    "gpu__time_duration.sum": "gpu__time_duration_us",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "smsp__issue_active.avg.pct": "issue_active_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1tex_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_scoreboard",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "stall_math_pipe",
}
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "msecond": 1e3, "usecond": 1.0,
        "nsecond": 1e-3, "ms": 1e3, "us": 1.0, "ns": 1e-3}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for i, n in enumerate(hdr):
        if n in WANT:
            v = float(vals[i].replace(",", ""))
            d[WANT[n]] = v * UNIT.get(units[i], 1.0) if units[i] in UNIT else v
    return d


rows = list(csv.reader(l for l in open(launches) if l.startswith('"')))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] += float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-3)
    cnt[name] += 1
# shares among the kernels of the wide engine's round loop (the launch list
# also holds the slot kernel's comparison runs, the decode and torch's fills)
ROUND = ("k_wide_dec", "k_wide_rows", "k_dd_step", "k_wide_compact", "k_wide_pack", "k_wide_bv", "k_fill")
total = sum(v for k, v in tot.items() if any(r in k for r in ROUND))
kernels = {k: {"launches": cnt[k], "device_ms": round(tot[k] / 1e3, 3),
               "share_of_round_loop": round(tot[k] / total, 4) if any(r in k for r in ROUND) else None}
           for k in sorted(tot, key=tot.get, reverse=True) if tot[k] / 1e3 > 0.05}
caps = [raw(r) for r in reps]
for c in caps:
    for k in kernels:
        if k.split("<")[0].replace("ddnm::", "") + "<" in c["kernel"]:
            kernels[k]["full_batch_launch"] = {a: b for a, b in c.items() if a != "kernel"}
dec = caps[0]
json.dump({
    "command": "bench.py --steps 1 --warmup 3 --no-cpu --no-subdomain --no-weak (launch list: every kernel of "
               "the run -- 6 wide solves of 40 rounds, the slot kernel's comparison runs, the decode; "
               "share_of_round_loop = of the wide engine's summed device time)",
    "dominant_kernel": dec["kernel"],
    "traffic_bytes_per_launch": dec["dram_bytes_read"] + dec["dram_bytes_write"],
    "kernels": kernels,
}, open(out, "w"), indent=1)
print(json.dumps(kernels, indent=1))
