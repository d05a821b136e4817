#!/usr/bin/env python3
"""Kernel timeline of bench.py's pipelined requests step as it runs now (scoring
of every batch on one stream with RTLM_SCORE_CTAS CTAs, each batch's schedule on
its slot's stream, depth 6), with torch.profiler; prints the scoring stream's
busy fraction, the mean scoring-kernel duration inside the pipeline and the
per-batch time.  Usage: python scripts/prof_pipe2.py out.json [K] [score_ctas]"""
import json
import os
import re
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_06619_b200 as rt  # noqa: E402
from rtgen import configs  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/pipe2.json"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 30
sc = int(sys.argv[3]) if len(sys.argv) > 3 else 70
part = os.environ.get("PIPE_PART", "all")  # "schedule": the batches are scored once, only schedules are timed
dev = torch.device("cuda", 0)
depth, n = int(os.environ.get("PIPE_DEPTH", "6")), 1 << 20
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
score_stream = torch.cuda.Stream(dev)
ev_scored = [torch.cuda.Event() for _ in ds]
ev_sched = [torch.cuda.Event() for _ in ds]
seg = np.asarray([0, n], np.uint32)
for c in ctxs:
    c.set_sm_limit(sc)
prof, reg = ds[0]["profile"], ds[0]["regressor"]


def step(k, score=None):
    sl = k % depth
    if score is None:
        score = part != "schedule"
    if score:
        with torch.cuda.stream(score_stream):
            score_stream.wait_event(ev_sched[sl])
            ctxs[sl].score_key(data[sl], off[sl], reg, prof, want_D=False, out=outs[sl])
            ev_scored[sl].record(score_stream)
    with torch.cuda.stream(streams[sl]):
        streams[sl].wait_event(ev_scored[sl])
        ctxs[sl].schedule(outs[sl]["key"], outs[sl]["u"], seg, prof, out=souts[sl])
        ev_sched[sl].record(streams[sl])


for k in range(2 * depth):
    step(k, True)
torch.cuda.synchronize()
import time  # noqa: E402
for rep in range(3):  # host issue cost of `depth` steps (well under the launch-queue capacity), GPU idle at the start
    h0 = time.perf_counter()
    for k in range(depth):
        step(k)
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"host issue: {(h1 - h0) * 1e3 / depth:.4f} ms per step")
if os.environ.get("PIPE_HOST"):  # per-call host time of the issue loop (no profiler)
    torch.cuda.synchronize()
    hs = []
    h0 = time.perf_counter()
    for k in range(K):
        a0 = time.perf_counter()
        step(k)
        hs.append((time.perf_counter() - a0) * 1e3)
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    h2 = time.perf_counter()
    print(f"{part}: issue loop {(h1 - h0) * 1e3 / K:.4f} ms per step, to completion {(h2 - h0) * 1e3 / K:.4f}; "
          f"per-call ms: " + " ".join(f"{x:.2f}" for x in hs))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as p:
    ev0.record()
    for st in streams + [score_stream]:
        st.wait_event(ev0)
    for k in range(K):
        step(k)
    for st in streams + [score_stream]:
        torch.cuda.current_stream().wait_stream(st)
    ev1.record()
    torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1) / K
p.export_chrome_trace(out)
tr = json.load(open(out))
ev = sorted((e for e in tr["traceEvents"] if e.get("cat") == "kernel"), key=lambda e: e["ts"])
sco = [e for e in ev if "k_score6" in e["name"]]
if not sco:
    print(f"{part} depth {depth}: {ms:.4f} ms/batch")
    sys.exit(0)
t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
busy = sum(e["dur"] for e in sco)
gaps = [b["ts"] - (a["ts"] + a["dur"]) for a, b in zip(sco, sco[1:])]
chain = [e for e in ev if "k_cpu_chain" in e["name"]]
print(f"score_ctas {sc}: {ms:.4f} ms/batch; span {(t1 - t0) / 1e3:.3f} ms; scoring kernels {len(sco)}, mean "
      f"{busy / len(sco):.1f} us, busy {busy / (t1 - t0):.3f} of the span, mean gap {np.mean(gaps):.1f} us "
      f"(max {max(gaps):.1f}); chain mean {np.mean([e['dur'] for e in chain]):.1f} us")
# what runs during the scoring gaps: kernels overlapping each gap, by name
cnt = {}
for a, b in zip(sco, sco[1:]):
    g0, g1 = a["ts"] + a["dur"], b["ts"]
    if g1 - g0 < 5:
        continue
    for e in ev:
        if e["ts"] < g1 and e["ts"] + e["dur"] > g0 and "k_score6" not in e["name"]:
            nm = re.sub(r"^void ", "", e["name"].replace("rtlm::(anonymous namespace)::", "")).split("(")[0][:30]
            cnt[nm] = cnt.get(nm, 0) + min(g1, e["ts"] + e["dur"]) - max(g0, e["ts"])
print("kernel-us overlapping the scoring gaps:", sorted(((round(v), k) for k, v in cnt.items()), reverse=True)[:10])
