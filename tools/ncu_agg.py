"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
ui = hdr.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    v *= {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(u, 1e-6)
    name = r[ki].split("(")[0]
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"{tot[k]:10.3f} ms {100*tot[k]/s:5.1f}%  n={cnt[k]:5d}  avg {1e3*tot[k]/cnt[k]:9.1f} us  {k}")
print(f"{s:10.3f} ms total")
