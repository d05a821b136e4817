#!/usr/bin/env python3
"""Runs rt_score_key on the config-2 queue a few times (for ncu captures of the scoring kernel, k_score6)
and prints the CUDA-event time per launch.  Usage: python scripts/prof_score.py [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_06619_b200 as rt  # noqa: E402
from rtgen import configs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
d = configs.config2()
dev = torch.device("cuda", 0)
ctx = rt.Context(d["lexicon"], 0)
data = torch.from_numpy(d["data"]).to(dev)
off = torch.from_numpy(d["offsets"].view(np.int32)).to(dev)
for _ in range(2):
    out = ctx.score_key(data, off, d["regressor"], d["profile"])
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = ctx.score_key(data, off, d["regressor"], d["profile"])
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("score_key ms:", " ".join(f"{t:.4f}" for t in ts), "min", f"{min(ts):.4f}")
