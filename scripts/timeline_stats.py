#!/usr/bin/env python3
"""Summarise a torch.profiler chrome trace of the pipelined step: wall span,
per-kernel total time, and per-kernel "exclusive" time (intervals during which
that kernel family is the only one running: the serial bottlenecks).
usage: timeline_stats.py trace.json"""
import collections
import json
import re
import sys

tr = json.load(open(sys.argv[1]))
ev = [e for e in tr["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = min(e["ts"] for e in ev)
t1 = max(e["ts"] + e["dur"] for e in ev)
name = lambda e: re.sub(r"^void ", "", e["name"].replace("rtlm::(anonymous namespace)::", "")).split("(")[0].split("<")[0][:40]  # noqa: E731
tot = collections.Counter()
cnt = collections.Counter()
for e in ev:
    tot[name(e)] += e["dur"]
    cnt[name(e)] += 1
# sweep: time with exactly one kernel running, attributed to it; and time with k running
pts = []
for i, e in enumerate(ev):
    pts.append((e["ts"], 1, i))
    pts.append((e["ts"] + e["dur"], -1, i))
pts.sort()
active = set()
excl = collections.Counter()
conc = collections.Counter()
last = pts[0][0]
for ts, d, i in pts:
    dt = ts - last
    if dt > 0:
        conc[len(active)] += dt
        if len(active) == 1:
            excl[name(ev[next(iter(active))])] += dt
    last = ts
    if d > 0:
        active.add(i)
    else:
        active.discard(i)
span = t1 - t0
print(f"span {span / 1e3:.3f} ms, kernels {len(ev)}")
print("concurrency (kernels running: share of span):",
      ", ".join(f"{k}: {v / span * 100:.1f}%" for k, v in sorted(conc.items())))
print(f"{'kernel':40s} {'n':>4s} {'total ms':>9s} {'mean us':>8s} {'alone ms':>9s}")
for k, v in tot.most_common(30):
    print(f"{k:40s} {cnt[k]:4d} {v / 1e3:9.3f} {v / cnt[k]:8.1f} {excl[k] / 1e3:9.3f}")
