#!/usr/bin/env python3
"""Coarse timeline of the pipelined requests step: CUDA events around each
batch's score_key and schedule calls on its stream (relative to one base
event), printed per batch.  Usage: python scripts/timeline.py [depth] [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_06619_b200 as rt  # noqa: E402
from rtgen import configs  # noqa: E402

dev = torch.device("cuda", 0)
depth = int(sys.argv[1]) if len(sys.argv) > 1 else 4
K = int(sys.argv[2]) if len(sys.argv) > 2 else 12
n = 1 << 20
ds = [configs.config2(n=n, gid0=i * n) for i in range(depth)]
ctxs = [rt.Context(d["lexicon"], 0) for d in ds]
data = [torch.from_numpy(d["data"]).to(dev) for d in ds]
off = [torch.from_numpy(d["offsets"].view(np.int32)).to(dev) for d in ds]
outs = [{"u": torch.empty(n, dtype=torch.float32, device=dev), "key": torch.empty(n, dtype=torch.int64, device=dev)} for _ in ds]
souts = [{"perm": torch.empty(n, dtype=torch.int32, device=dev), "batch_of": torch.empty(n, dtype=torch.int32, device=dev),
          "slot_of": torch.empty(n, dtype=torch.uint8, device=dev), "core_of": torch.empty(n, dtype=torch.uint8, device=dev),
          "seg_batch_off": torch.empty(2, dtype=torch.int32, device=dev)} for _ in ds]
streams = [torch.cuda.Stream(dev) for _ in ds]
seg = np.asarray([0, n], np.uint32)
for c in ctxs:
    c.set_sm_limit(148 - depth)
prof, reg = ds[0]["profile"], ds[0]["regressor"]
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def step(k, ev=None):
    sl = k % depth
    with torch.cuda.stream(streams[sl]):
        if ev: ev[0].record()
        ctxs[sl].score_key(data[sl], off[sl], reg, prof, want_D=False, out=outs[sl])
        if ev: ev[1].record()
        ctxs[sl].schedule(outs[sl]["key"], outs[sl]["u"], seg, prof, out=souts[sl])
        if ev: ev[2].record()


for k in range(2 * depth):
    step(k)
torch.cuda.synchronize()
base = E()
base.record()
for st in streams:
    st.wait_event(base)
evs = [[E(), E(), E()] for _ in range(K)]
for k in range(K):
    step(k, evs[k])
torch.cuda.synchronize()
for k in range(K):
    a, b, c = (base.elapsed_time(e) for e in evs[k])
    print(f"batch {k:2d} slot {k % depth}: score {a:7.3f} -> {b:7.3f} ({b - a:.3f})  schedule -> {c:7.3f} ({c - b:.3f})")
