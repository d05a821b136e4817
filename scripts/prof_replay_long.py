#!/usr/bin/env python3
"""rt_simulate on full paper-length traces (the beta = 10..150 ramp, 11 280
arrivals each; k_replay_long), 148 traces x 4 LMs; CUDA-event ms.
Usage: python scripts/prof_replay_long.py [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_06619_b200 as rt  # noqa: E402
from rtgen import configs  # noqa: E402
import bench  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda", 0)
nt = 148
d = configs.traces(3, range(30000, 30000 + nt), 11280, lambda t: (t - 30000) * 4 // nt)
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
print(f"long replay: {nt} traces x 11280, ms min {min(ts):.3f} -> {nt / (min(ts) / 1e3):.0f} traces/s")
