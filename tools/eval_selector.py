"""Score the selector AS THE LIBRARY RUNS IT (H2 / f2; the paper's Fig. 6
analog): for every workload of the performance database, call
libgeot's geot_select_config_ex (through ctypes, pure host — no GPU needed)
with the workload's real skew and with skew unknown, and geot_select_hand_rules
for the pre-refit baseline; look the chosen configurations up in the measured
times.  Quality = geomean over workloads of best measured time / time of the
selected configuration (1.0 = always the best).  A selected configuration the
database never timed is reported, never guessed.

    python tools/eval_selector.py profiles/perfdb_r2.jsonl [--report profiles/selector_report_r2.md]
"""
from __future__ import annotations

import argparse
import ctypes
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import refit_selector as R  # noqa: E402
from paper_2404_03019_b200 import _lib  # noqa: E402

OPS = {"sum": 0, "mean": 1, "max": 2}


def label_of(c):
    return R.label({"variant": c.variant, "rows_per_group": c.rows_per_group, "warps_per_cta": c.warps_per_cta,
                    "stages": c.stages})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("db", nargs="+")
    ap.add_argument("--report")
    a = ap.parse_args()
    L = _lib.load()
    by = R.build(R.load(a.db))
    keys = sorted(by)
    rows = []
    for k in keys:
        E, S, F, dt, dist, fused, op = k[:7]
        times = by[k]
        best_lab = min(times, key=times.get)
        best = times[best_lab]
        ml = R.MAXLEN.get(k) or 0
        skew = ml / (E / max(S, 1)) if ml else 0.0
        res = {}
        for name, fn in (("known", lambda c: L.geot_select_config_ex(E, S, F, OPS[op], 0 if dt == "f32" else 1, 0,
                                                                     int(fused), skew, ctypes.byref(c))),
                         ("unknown", lambda c: L.geot_select_config_ex(E, S, F, OPS[op], 0 if dt == "f32" else 1, 0,
                                                                       int(fused), 0.0, ctypes.byref(c))),
                         ("hand", lambda c: L.geot_select_hand_rules(E, S, F, 0 if dt == "f32" else 1, int(fused),
                                                                     ctypes.byref(c)))):
            c = _lib.GeotConfig()
            assert fn(c) == 0
            lab = label_of(c)
            res[name] = (lab, times.get(lab))
        rows.append((k, best_lab, best, res, R.is_test(k)))

    def quality(sel, name):
        r = [best / res[name][1] for (_k, _bl, best, res, _t) in sel if res[name][1] is not None]
        missing = sum(1 for (_k, _bl, _b, res, _t) in sel if res[name][1] is None)
        return (float(np.exp(np.mean(np.log(r)))) if r else float("nan")), missing, len(r)

    splits = {"held-out": [r for r in rows if r[4]], "train": [r for r in rows if not r[4]], "all": rows}
    lines = ["| split | workloads | library, skew known | library, skew unknown | hand rules |", "|---|---|---|---|---|"]
    for sname, sel in splits.items():
        cells = []
        for name in ("known", "unknown", "hand"):
            q, miss, n = quality(sel, name)
            cells.append(f"{q:.3f}" + (f" ({miss} untimed)" if miss else ""))
        lines.append(f"| {sname} | {len(sel)} | " + " | ".join(cells) + " |")
    table = "\n".join(lines)
    print(table)
    prov = L.geot_selector_provenance().decode()
    if a.report:
        with open(a.report, "w") as f:
            f.write("# Selector quality as the library selects (H2 / f2; PAPER.md §III-C P:301-315, Fig. 6 "
                    "analog P:459-462)\n\n")
            f.write(f"- compiled tree: {prov}\n")
            f.write(f"- perf DB: {', '.join(os.path.basename(d) for d in a.db)}; {len(keys)} workloads, "
                    f"{sum(len(v) for v in by.values())} (workload, configuration) timings\n")
            f.write("- scored by calling libgeot's `geot_select_config_ex` (ctypes) with each workload's real "
                    "skew (max segment length / avg) and with skew unknown (the cfg=NULL path), and "
                    "`geot_select_hand_rules` for the pre-refit baseline; a selection the database never timed "
                    "is counted as untimed, not guessed\n")
            f.write("- quality = geomean over workloads of best measured time / time of the selected configuration\n\n")
            f.write(table + "\n\n")
            f.write("## Held-out workloads\n\n| E | S | F | dtype | dist | fused | op | tag | skew | best | us | "
                    "library (known skew) | us | hand rules | us |\n|" + "---|" * 15 + "\n")
            for (k, bl, best, res, t) in rows:
                if not t:
                    continue
                E, S = k[0], k[1]
                ml = R.MAXLEN.get(k) or 0
                sk = ml / (E / max(S, 1)) if ml else float("nan")
                kl, kt = res["known"]
                hl, ht = res["hand"]
                f.write(f"| {k[0]} | {k[1]} | {k[2]} | {k[3]} | {k[4]} | {k[5]} | {k[6]} | {k[7]} | {sk:.0f} | {bl} | "
                        f"{best * 1e3:.1f} | {kl} | {'untimed' if kt is None else f'{kt * 1e3:.1f}'} | {hl} | "
                        f"{'untimed' if ht is None else f'{ht * 1e3:.1f}'} |\n")


if __name__ == "__main__":
    main()
