#!/usr/bin/env python3
"""rt_predict_mlp on config-2 features (random-init weights): CUDA-event ms per launch.
Usage: python scripts/prof_mlp.py [reps] [fp32|bf16]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_06619_b200 as rt  # noqa: E402
import rtgen  # noqa: E402
from rtgen import configs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
d = configs.config2()
dev = torch.device("cuda", 0)
ctx = rt.Context(d["lexicon"], 0)
feat = ctx.score(torch.from_numpy(d["data"]).to(dev), torch.from_numpy(d["offsets"].view(np.int32)).to(dev))
ws, bs = rtgen.mlp_weights(12345)
ctx.set_mlp(ws, bs)
ctx.set_mlp_precision(sys.argv[2] if len(sys.argv) > 2 else "bf16")
u = torch.empty(feat.shape[0], dtype=torch.float32, device=dev)
for _ in range(3):
    ctx.predict_mlp(feat, u)
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.predict_mlp(feat, u)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("mlp ms min", f"{min(ts):.4f}", "median", f"{sorted(ts)[len(ts) // 2]:.4f}")
if os.environ.get("KTF_TRACE"):
    print("trace", [int(x) for x in u[:16].cpu().tolist()])
