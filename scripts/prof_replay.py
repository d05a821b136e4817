#!/usr/bin/env python3
"""Runs rt_score_key + rt_simulate on the config-3 traces (4096 x 1000, 4 LMs) a few
times (for ncu captures of k_replay) and prints the CUDA-event time of the replay.
Usage: python scripts/prof_replay.py [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_06619_b200 as rt  # noqa: E402
from rtgen import configs  # noqa: E402
import bench  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda", 0)
nt = 4096
d = configs.traces(3, range(nt), 1000, lambda t: (t // (nt // 4)) % 4)
ctx = rt.Context(d["lexicon"], 0)
n = len(d["arrival_us"])
arr = torch.from_numpy(d["arrival_us"]).to(dev)
tl = torch.from_numpy(d["true_len"].view(np.int16)).to(dev)
tp = torch.from_numpy(d["trace_prof"].view(np.int16)).to(dev)
u = torch.empty(n, dtype=torch.float32, device=dev)
key = torch.empty(n, dtype=torch.int64, device=dev)
D = torch.empty(n, dtype=torch.int32, device=dev)
for f, r0, r1, gd, so in bench._lm_groups(d, dev):
    ctx.score_key(gd, so, d["regressors"][f], d["profiles"][f], arrival=arr[r0:r1],
                  out={"u": u[r0:r1], "key": key[r0:r1], "D": D[r0:r1]})
stats = torch.empty((nt, 2), dtype=torch.int64, device=dev)
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.simulate(arr, tl, u, key, D, d["trace_off"], d["profiles"], tp, stats=stats)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("replay ms:", " ".join(f"{t:.4f}" for t in ts), "min", f"{min(ts):.4f}")
