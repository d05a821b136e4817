#!/usr/bin/env python3
"""Per-source-line warp instructions per loop iteration of k_score5 from an
ncu report: python scripts/k5_lines.py <report.ncu-rep> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]
tot, votes = 0, []
stalls = collections.Counter()
for r in rows[2:]:
    d = dict(zip(hdr, r))
    try:
        e = int(d["Instructions Executed"])
    except (KeyError, ValueError):
        continue
    tot += e
    if "VOTE.ANY" in d["Source"]:
        votes.append(e)
    for k, v in d.items():
        if k.startswith("stall_") and "(Not" not in k:
            try:
                stalls[k] += float(v)
            except ValueError:
                pass
it = max(votes) if votes else 1
print(f"total warp inst {tot / 1e6:.1f}M, loop iterations {it}, per iteration {tot / it:.1f}")
s = sum(stalls.values()) or 1
print("stalls:", ", ".join(f"{k[6:]} {v / s * 100:.1f}%" for k, v in stalls.most_common(8)))
cs = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                    capture_output=True, text=True).stdout
hdr = cur = None
agg = {}
for r in csv.reader(io.StringIO(cs)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            ie = float(d["Instructions Executed"] or 0)
            te = float(d["Thread Instructions Executed"] or 0)
        except (KeyError, ValueError):
            continue
        if ie:
            agg[(cur, int(r[0]))] = (ie, te, r[1][:90])
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / it:6.1f}/it act {v[1] / v[0]:4.1f} {k[0]}:{k[1]} {v[2]}")
