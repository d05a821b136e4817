#!/usr/bin/env python3
"""One rt_score_key + rt_schedule of the config-2 queue (for ncu per-kernel
SM-activity of the schedule).  Usage: python scripts/prof_sched.py [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_06619_b200 as rt  # noqa: E402
from rtgen import configs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
d = configs.config2()
dev = torch.device("cuda", 0)
ctx = rt.Context(d["lexicon"], 0)
data = torch.from_numpy(d["data"]).to(dev)
off = torch.from_numpy(d["offsets"].view(np.int32)).to(dev)
seg = np.asarray([0, len(d["offsets"]) - 1], np.uint32)
for _ in range(reps):
    out = ctx.score_key(data, off, d["regressor"], d["profile"])
    ctx.schedule(out["key"], out["u"], seg, d["profile"])
torch.cuda.synchronize()
