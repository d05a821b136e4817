#!/usr/bin/env python3
"""Warp instructions and stall samples of round-1 k_score4 grouped by phase (its k_score.cu line ranges; for k_score6 use ncu_ranges.py), from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv`.  usage: ncu_phases.py <csv>
Lines of other files (inlined intrinsics, internal.cuh helpers) are reported per file."""
import csv
import sys

PHASES = [("lexicon probe (lookup / word_code)", 82, 139), ("stage_run (clitic split)", 411, 437),
          ("flush_counts (atomics)", 544, 554), ("rules_round", 556, 632), ("task setup", 634, 702),
          ("(1) stage + classify", 703, 743), ("(2) events", 744, 804), ("(3) tokens", 805, 874),
          ("rule-round trigger", 875, 880), ("dropped bytes", 881, 889), ("chunk tail", 890, 897),
          ("epilogue", 898, 911), ("regress / key", 22, 68), ("fsm fallback", 146, 278), ("other", 0, 10 ** 9)]

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
    if cur != "k_score.cu":
        a = agg.setdefault("[" + cur + "]", [0.0, 0.0, 0.0])
        a[0] += ie
        a[1] += te
        a[2] += st
        continue
    key = ln
    for name, lo, hi in PHASES:
        if lo <= key <= hi:
            a = agg.setdefault(name, [0.0, 0.0, 0.0])
            a[0] += ie
            a[1] += te
            a[2] += st
            break
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[2] for v in agg.values()) or 1
print(f"total warp instructions {ti / 1e6:.1f} M")
for name, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {name:38s} {v[0] / 1e6:7.1f} M ({v[0] / ti * 100:4.1f} %)  lanes {v[1] / max(v[0], 1):5.1f}  "
          f"stall samples {v[2] / ts * 100:4.1f} %")
