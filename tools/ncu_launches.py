"""Summarise an ncu launch list (gpu__time_duration.sum per launch):
per-kernel count, mean time and share of the library's (geot::) launches.
Usage: python tools/ncu_launches.py launches.csv [--only geot::]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else "geot::"
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = defaultdict(list)
order = []
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    agg[name].append(float(r[vi]) / 1000.0)
    order.append(name)
tot = sum(sum(v) for k, v in agg.items() if only in k)
print(f"{'kernel':<72} {'launches':>8} {'mean us':>9} {'share of ' + only:>16}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    share = 100 * sum(v) / tot if only in k and tot else float("nan")
    print(f"{k[:72]:<72} {len(v):>8} {sum(v) / len(v):>9.2f} {share:>15.1f}%")
