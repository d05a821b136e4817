#!/usr/bin/env python3
"""Shared-memory wavefronts (and the excess over ideal) per source line, top N.
usage: ncu_smem_lines.py <src.csv> [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
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
        w = float(d.get("L1 Wavefronts Shared") or 0)
        wi = float(d.get("L1 Wavefronts Shared Ideal") or 0)
    except ValueError:
        continue
    a = agg.setdefault((cur, ln), [0.0, 0.0, r[1][:80]])
    a[0] += w
    a[1] += wi
tw = sum(v[0] for v in agg.values()) or 1
print(f"total shared wavefronts {tw / 1e6:.1f} M")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / 1e6:7.2f}M ({v[0] / tw * 100:4.1f}%) ideal {v[1] / 1e6:6.2f}M  {k[0]}:{k[1]:<5d} {v[2]}")
