"""Merge performance databases: records of a later file REPLACE every record of
the same workload (E, S, F, dtype, dist, fused, op) from earlier files, so the
configurations of one workload are always compared within one sweep (one box).

    python tools/merge_perfdb.py base.jsonl supplement.jsonl [...] > merged.jsonl
"""
import json
import sys


def wkey(r):
    return (r["E"], r["S"], r["F"], r["dtype"], r["dist"], r["fused"], r["op"])


def main():
    by = {}
    for path in sys.argv[1:]:
        recs = [json.loads(l) for l in open(path) if l.strip()]
        fresh = {}
        for r in recs:
            fresh.setdefault(wkey(r), []).append(r)
        by.update(fresh)
    for k in by:
        for r in by[k]:
            print(json.dumps(r))


if __name__ == "__main__":
    main()
