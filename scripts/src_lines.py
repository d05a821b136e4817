#!/usr/bin/env python3
"""Instruction counts per source line range of k_score.cu from an ncu source-page CSV.
usage: src_lines.py <csv> [lo hi]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur = None
hdr = None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        agg[(cur, ln)] = agg.get((cur, ln), [0, r[1]])
        agg[(cur, ln)][0] += float(d.get("Instructions Executed") or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values())
print(f"total {tot / 1e6:.1f} M warp-inst")
if len(sys.argv) > 3:
    lo, hi = int(sys.argv[2]), int(sys.argv[3])
    s = 0
    for (f, l), v in sorted(agg.items()):
        if f == "k_score.cu" and lo <= l <= hi and v[0]:
            s += v[0]
            print(f"{l:5d} {v[0] / 1e6:7.2f}M  {v[1][:90]}")
    print(f"range {s / 1e6:.1f} M = {s / tot * 100:.1f}%")
