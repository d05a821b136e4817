#!/usr/bin/env python3
"""Warp instructions / active lanes / stall samples per k_score.cu line range.
usage: ncu_ranges.py <src.csv> name:lo-hi [name:lo-hi ...]   (other files and lines -> 'other')"""
import csv
import sys

ranges = []
for a in sys.argv[2:]:
    name, rng = a.split(":")
    lo, hi = rng.split("-")
    ranges.append((name, int(lo), int(hi)))
rows = list(csv.reader(open(sys.argv[1], errors="replace")))
cur = hdr = None
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
    d = dict(zip(hdr, r))
    try:
        ie = float(d.get("Instructions Executed") or 0)
        te = float(d.get("Thread Instructions Executed") or 0)
        st = float(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        continue
    name = "other [" + str(cur) + "]"
    if cur == "k_score.cu":
        for nm, lo, hi in ranges:
            if lo <= ln <= hi:
                name = nm
                break
    a = agg.setdefault(name, [0.0, 0.0, 0.0])
    a[0] += ie
    a[1] += te
    a[2] += st
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[2] for v in agg.values()) or 1
print(f"total warp instructions {ti / 1e6:.1f} M")
for name, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {name:34s} {v[0] / 1e6:7.1f} M ({v[0] / ti * 100:4.1f} %)  lanes {v[1] / max(v[0], 1):5.1f}  "
          f"stall {v[2] / ts * 100:4.1f} %")
