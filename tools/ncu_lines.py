"""Aggregate an ncu source page (cuda,sass csv) per CUDA source line:
instructions executed and stall samples.  Usage:
  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
  python tools/ncu_lines.py src.csv [topN]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(lambda: [0, 0, ""])
fname = ""
cur_line = None
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0].strip():
        cur_line = (fname, int(r[0]))
        agg[cur_line][2] = r[1].strip()[:80]
    if cur_line is None:
        continue
    try:
        ie = int(r[7] or 0)
        ns = int(r[6] or 0)
    except ValueError:
        continue
    agg[cur_line][0] += ie
    agg[cur_line][1] += ns
tot_i = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values())
print(f"total instructions {tot_i}  samples {tot_s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]}:{k[1]:<5} inst {v[0]:>10} ({100*v[0]/max(tot_i,1):5.1f}%) samples {v[1]:>6} ({100*v[1]/max(tot_s,1):5.1f}%)  {v[2]}")
