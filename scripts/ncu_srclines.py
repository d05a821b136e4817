#!/usr/bin/env python3
"""Per-source-line warp instructions, active threads and stall samples from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`.
usage: ncu_srclines.py <csv> [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
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
    if r[0] == "Function Name" or hdr is None:
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
    a = agg.setdefault((cur, ln), [0.0, 0.0, 0.0, r[1][:90]])
    a[0] += ie
    a[1] += te
    a[2] += st
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[2] for v in agg.values()) or 1
print(f"total warp inst {ti / 1e6:.1f}M")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
    print(f"{v[2] / ts * 100:5.1f}% stall {v[0] / ti * 100:5.1f}% inst act {v[1] / max(v[0], 1):5.1f} {k[0]}:{k[1]:<4d} {v[3]}")
