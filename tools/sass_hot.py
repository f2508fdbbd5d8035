"""Summarise an ncu source-page CSV (--page source --csv --print-source sass):
the hot SASS (executed >= frac * max) in address order with exec counts and
stall samples, plus totals per opcode.  python tools/sass_hot.py X.csv[.gz] [frac]"""
import csv
import gzip
import io
import sys
from collections import Counter

path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
lines = raw.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
ex = [int(r["Instructions Executed"] or 0) for r in rows]
mx = max(ex)
tot = sum(ex)
samp = [int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows]
print(f"total warp instructions {tot:,}; samples {sum(samp):,}")
ops = Counter()
for r, e in zip(rows, ex):
    op = r["Source"].strip().split()[0] if r["Source"].strip() else "?"
    if op.startswith("@"):
        op = r["Source"].strip().split()[1]
    ops[op.split(".")[0]] += e
print("by opcode:", ", ".join(f"{k} {v / tot:.1%}" for k, v in ops.most_common(25)))
for r, e, s in zip(rows, ex, samp):
    if e >= frac * mx or s >= 0.01 * sum(samp):
        print(f"{r['Address'][-5:]} {e:>12,} {s:>6} {r['Source'].strip()[:90]}")
