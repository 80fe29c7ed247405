"""Aggregate ncu warp-stall samples per CUDA source line from `ncu -i rep --page source --csv
--print-source cuda,sass` output.  python tools/ncu_source_lines.py <csv> [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(lambda: [0.0, 0.0, ""])
fname = "?"
hdr = None
cur = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 6:
        continue
    if r[0]:
        cur = (fname, r[0], r[1].strip()[:80])
    if cur is None:
        continue
    iS = 4
    try:
        agg[cur][0] += float(r[iS] or 0)
        agg[cur][1] += float(r[7] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values())
print(f"total samples {tot:.0f}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}% {v[1]:>10.0f}  {k[0]}:{k[1]}  {k[2]}")
