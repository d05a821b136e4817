#!/usr/bin/env python3
"""Per-source-line totals from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = None
agg = {}
hdr = None
for row in csv.reader(open(path)):
    if not row:
        continue
    if row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or row[0] in ("Function Name",):
        continue
    d = dict(zip(hdr[2:], row[2:]))
    try:
        line = int(row[0])
    except ValueError:
        continue
    key = (cur_file, line)
    a = agg.setdefault(key, [0.0, 0.0, row[1][:100]])
    try:
        a[0] += float(d.get("Warp Stall Sampling (All Samples)") or 0)
        a[1] += float(d.get("Instructions Executed") or 0)
    except ValueError:
        pass
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[1] / ti * 100:5.1f}% inst {v[0] / ts * 100:5.1f}% stall  {k[0]}:{k[1]:<5d} {v[2]}")
