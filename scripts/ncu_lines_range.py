#!/usr/bin/env python3
"""Per-line warp instructions of k_score.cu lines lo..hi.  usage: ncu_lines_range.py <src.csv> lo hi"""
import csv
import sys

lo, hi = int(sys.argv[2]), int(sys.argv[3])
rows = list(csv.reader(open(sys.argv[1], errors="replace")))
cur = hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or cur != "k_score.cu":
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    if not lo <= ln <= hi:
        continue
    d = dict(zip(hdr, r))
    try:
        ie = float(d.get("Instructions Executed") or 0)
        te = float(d.get("Thread Instructions Executed") or 0)
    except ValueError:
        continue
    print(f"{ln:5d} {ie / 1e6:7.2f}M lanes {te / max(ie, 1):5.1f}  {r[1][:110]}")
