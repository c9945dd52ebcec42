"""Aggregate ncu source-page warp-stall samples per CUDA source line.

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > f.csv
       python tools/ncu_lines.py f.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = None
hdr = None
stats = []
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        samp = int(r[4] or 0)
    except ValueError:
        continue
    d = dict(zip(hdr[4:], r[4:]))
    stall = {k: d[k] for k in d if k.startswith("stall_") and "Not Issued" not in k and d[k] not in ("", "0")}
    stats.append((samp, cur_file, r[0], r[1][:90], stall))
tot = sum(s[0] for s in stats)
stats.sort(key=lambda s: -s[0])
print("total samples", tot)
for s in stats[:top]:
    st = sorted(((int(v), k[6:]) for k, v in s[4].items() if v.isdigit()), reverse=True)[:3]
    print(f"{100*s[0]/tot:5.1f}% {s[1]}:{s[2]:>4} {s[3]:<90} {st}")
