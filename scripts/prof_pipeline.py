#!/usr/bin/env python3
"""Kernel timeline of the pipelined requests step (bench.py's depth-4 leg) with
torch.profiler (CUPTI activity records: per-kernel start / end / stream), for
finding what bounds the step.  Usage: python scripts/prof_pipeline.py out.json [K]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_06619_b200 as rt  # noqa: E402
from rtgen import configs  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/pipe_trace.json"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 16
part = os.environ.get("RTLM_BENCH_PART", "all")
dev = torch.device("cuda", 0)
depth = 4
n = 1 << 20
ds = [configs.config2(n=n, gid0=i * n) for i in range(depth)]
ctxs = [rt.Context(d["lexicon"], 0) for d in ds]
data = [torch.from_numpy(d["data"]).to(dev) for d in ds]
off = [torch.from_numpy(d["offsets"].view(np.int32)).to(dev) for d in ds]
outs = [{"u": torch.empty(n, dtype=torch.float32, device=dev), "key": torch.empty(n, dtype=torch.int64, device=dev)}
        for _ in ds]
souts = [{"perm": torch.empty(n, dtype=torch.int32, device=dev), "batch_of": torch.empty(n, dtype=torch.int32, device=dev),
          "slot_of": torch.empty(n, dtype=torch.uint8, device=dev), "core_of": torch.empty(n, dtype=torch.uint8, device=dev),
          "seg_batch_off": torch.empty(2, dtype=torch.int32, device=dev)} for _ in ds]
streams = [torch.cuda.Stream(dev) for _ in ds]
seg = np.asarray([0, n], np.uint32)
nsm = torch.cuda.get_device_properties(dev).multi_processor_count
for c in ctxs:
    c.set_sm_limit(nsm - depth)
prof, reg = ds[0]["profile"], ds[0]["regressor"]


def step(k):
    sl = k % depth
    with torch.cuda.stream(streams[sl]):
        if part in ("all", "score"):
            ctxs[sl].score_key(data[sl], off[sl], reg, prof, want_D=False, out=outs[sl])
        if part in ("all", "schedule"):
            ctxs[sl].schedule(outs[sl]["key"], outs[sl]["u"], seg, prof, out=souts[sl])


for k in range(2 * depth):
    step(k)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as p:
    ev0.record()
    for st in streams:
        st.wait_event(ev0)
    for k in range(K):
        step(k)
    for st in streams:
        torch.cuda.current_stream().wait_stream(st)
    ev1.record()
    torch.cuda.synchronize()
print(f"{part}: {ev0.elapsed_time(ev1) / K:.4f} ms per batch")
p.export_chrome_trace(out)
