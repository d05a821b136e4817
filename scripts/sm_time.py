#!/usr/bin/env python3
"""Per-kernel duration and SM-active time (as microseconds of the whole GPU)
from an ncu --csv launch list with gpu__time_duration.sum and
sm__cycles_active.sum; the second half of the launches (the warm rep).
usage: sm_time.py <csv> [sm_mhz]"""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read().splitlines()
clk = float(sys.argv[2]) * 1e6 if len(sys.argv) > 2 else 1.965e9
i = [k for k, l in enumerate(txt) if l.startswith('"ID"')][0]
by = collections.OrderedDict()
for r in csv.DictReader(io.StringIO("\n".join(txt[i:]))):
    name = r["Kernel Name"].split("(")[0].replace("rtlm::(anonymous namespace)::", "").replace("void ", "")
    by.setdefault((r["ID"], name[:34]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
items = list(by.items())[len(by) // 2:]
agg = collections.OrderedDict()
for (_, name), m in items:
    a = agg.setdefault(name, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0) / 1e3
    a[2] += m.get("sm__cycles_active.sum", 0) / clk * 1e6 / 148
tot = sum(a[2] for a in agg.values())
print(f"{'kernel':34s} {'n':>3s} {'us':>8s} {'GPU-us':>8s}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][2]):
    print(f"{k:34s} {a[0]:3d} {a[1]:8.1f} {a[2]:8.1f}")
print(f"total GPU-us (SM-active / 148 SMs): {tot:.1f}")
