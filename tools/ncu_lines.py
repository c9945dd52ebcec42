"""Aggregate an ncu source page (CUDA lines with their SASS) per source line
and per enclosing function.

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > f.csv
       python tools/ncu_lines.py f.csv [top]"""
import csv
import os
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = None
hdr = None
stats = []
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    d = dict(zip(hdr[4:], r[4:]))

    def num(k):
        try:
            return int(d.get(k, "0") or 0)
        except ValueError:
            return 0
    stall = {k: num(k) for k in d if k.startswith("stall_") and "Not Issued" not in k}
    stats.append(dict(samp=num("Warp Stall Sampling (All Samples)"),
                      inst=num("Instructions Executed"), file=cur_file, line=int(r[0]),
                      src=r[1].strip()[:80], stall=stall))

# enclosing function of each line: nearest preceding definition-looking line
func_starts = {}
for f in {s["file"] for s in stats}:
    starts = []
    if f and os.path.exists(f):
        for i, ln in enumerate(open(f), 1):
            m = re.match(r"^(?:template <[^>]*>\s*)?(?:static\s+)?(?:__device__|__global__)[^(]*?\b(\w+)\s*\(", ln)
            if m:
                starts.append((i, m.group(1)))
    func_starts[f] = starts


def func_of(s):
    name = "?"
    for i, n in func_starts.get(s["file"], []):
        if i <= s["line"]:
            name = n
    return os.path.basename(s["file"] or "?") + ":" + name


tot = sum(s["samp"] for s in stats) or 1
toti = sum(s["inst"] for s in stats) or 1
agg = {}
for s in stats:
    a = agg.setdefault(func_of(s), [0, 0])
    a[0] += s["samp"]
    a[1] += s["inst"]
print(f"total samples {tot}, warp instructions {toti}")
print("-- per function (samples %, instructions %)")
for k, (sa, ins) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{100 * sa / tot:5.1f}% {100 * ins / toti:5.1f}%  {k}")
print("-- top lines")
stats.sort(key=lambda s: -s["samp"])
for s in stats[:top]:
    st = sorted(((v, k[6:]) for k, v in s["stall"].items() if v), reverse=True)[:3]
    print(f"{100 * s['samp'] / tot:5.1f}% {100 * s['inst'] / toti:5.1f}% "
          f"{os.path.basename(s['file'] or '?')}:{s['line']:>4} {s['src']:<80} {st}")
