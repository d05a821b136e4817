#!/usr/bin/env python3
"""Host-side issue time of the pipelined requests step (is the bench host-bound?).
Times enqueueing K score_key+schedule steps (no sync) vs the device time."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_06619_b200 as rt  # noqa: E402
from rtgen import configs  # noqa: E402

dev = torch.device("cuda", 0)
depth, K = 4, 40
ds = [configs.config2(n=1 << 20, gid0=i << 20) for i in range(depth)]
ctxs = [rt.Context(d["lexicon"], 0) for d in ds]
data = [torch.from_numpy(d["data"]).to(dev) for d in ds]
off = [torch.from_numpy(d["offsets"].view(np.int32)).to(dev) for d in ds]
n = 1 << 20
outs = [{"u": torch.empty(n, dtype=torch.float32, device=dev), "key": torch.empty(n, dtype=torch.int64, device=dev)} for _ in ds]
souts = [{"perm": torch.empty(n, dtype=torch.int32, device=dev), "batch_of": torch.empty(n, dtype=torch.int32, device=dev),
          "slot_of": torch.empty(n, dtype=torch.uint8, device=dev), "core_of": torch.empty(n, dtype=torch.uint8, device=dev),
          "seg_batch_off": torch.empty(2, dtype=torch.int32, device=dev)} for _ in ds]
streams = [torch.cuda.Stream(dev) for _ in ds]
seg = np.asarray([0, n], np.uint32)
for c in ctxs:
    c.set_sm_limit(148 - depth)
prof, reg = ds[0]["profile"], ds[0]["regressor"]


def step(k, part):
    sl = k % depth
    with torch.cuda.stream(streams[sl]):
        if part in ("all", "score"):
            ctxs[sl].score_key(data[sl], off[sl], reg, prof, want_D=False, out=outs[sl])
        if part in ("all", "schedule"):
            ctxs[sl].schedule(outs[sl]["key"], outs[sl]["u"], seg, prof, out=souts[sl])


for part in ("score", "schedule", "all"):
    for k in range(8):
        step(k, part)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        step(k, part)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{part:9s} host issue {(t1 - t0) / K * 1e3:.3f} ms/step, wall {(t2 - t0) / K * 1e3:.3f} ms/step")
