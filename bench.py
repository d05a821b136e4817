#!/usr/bin/env python3
"""Benchmark of the RT-LM hot path on B200 (BASELINE.json metric:
"M requests scored+scheduled/s and traces/s at 1/2/4/8 B200; % of HBM peak").

One STEP = one pass of the hot path over one batch of synthetic input:
  * value (requests leg, BASELINE configs[1] = config 2): one queue of 2^20
    requests per GPU -> rt_score_key (a1-a4: features, u, key) -> rt_schedule
    (a5-a6: order, consolidation, CPU cores).  value = requests/s (whole job).
  * traces leg (configs[2] = config 3): 4096 Poisson traces x 1000 requests per
    GPU -> rt_score_key per LM (a1-a4) -> rt_simulate (a5 in-kernel sort, a6
    consolidation rounds, a7 replay) -> rt_reduce_stats + NCCL all-reduce (a8).
    Reported as traces/s in "traces".
Under torchrun each rank runs its own queue / trace shard (replicas / weak
scaling; the only collective is the int64 stats all-reduce).

L2 hygiene: the inputs of one requests step are ~100 MB (< 126 MB L2), so a
256 MB buffer is written between timed steps (outside the events).  Timing:
CUDA events on the launching stream around every step, summed; max over ranks.

--impl reference: the CPU oracle (oracle/, single thread) on a bounded sample
of the same workload, same metric/unit (the task's reference arm).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# The pipelined step runs 2 x depth + 1 streams (slot streams, the library's
# CPU-class fork streams, the scoring stream).  With the default 8 hardware
# work queues, streams share queues and their kernels wait on each other in
# submission order (false dependencies): the schedules of different batches
# then ran one after another (0.45 -> 0.25 ms per batch for schedules alone,
# pipelined step 0.59 -> 0.45 ms with 32 queues, profiles/notes/r02_schedule_pipeline.md).
# Read when the CUDA context is created, so it is set before torch touches CUDA.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

METRIC = "M requests scored+scheduled/s"
UNIT = "Mreq/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # 100 steps by default: the timed region holds the pipeline's fill and the
    # last batch's schedule (~2 ms, CPU-class-chain bound), which 40 steps
    # amortise to ~50 µs per step and 100 steps to ~20
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--n", type=int, default=1 << 20, help="requests per GPU queue (config 2)")
    ap.add_argument("--traces", type=int, default=4096, help="traces per GPU (config 3)")
    ap.add_argument("--per-trace", type=int, default=1000)
    ap.add_argument("--no-traces", action="store_true")
    ap.add_argument("--no-mlp", action="store_true")
    ap.add_argument("--sweeps", action="store_true", help="also run the NEXT-3 malicious-ratio sweep")
    ap.add_argument("--no-config4", action="store_true",
                    help="skip config 4: 65536 traces x 1024 (2^26 requests) split over the ranks (strong scaling)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only: run the N-rank plumbing (self-spawn, gloo init, config-4 block shards, int64 SUM "
                         "all-reduce, MAX-over-ranks timing, rank-0 JSON line) without any kernel; for tests")
    ap.add_argument("--no-config5", action="store_true", help="skip config 5 (rate/deadline x ablation sweep)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--depth", type=int, default=8, help="batches in flight (contexts / streams / distinct inputs)")
    ap.add_argument("--graphs", action="store_true",
                    help="replay one CUDA graph per batch slot instead of issuing the pipelined step call by call")
    return ap.parse_args()


def dist_env():
    from paper_2309_06619_b200 import dist as rdist
    return rdist.env()


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(args) -> int:
    """`--gpus N` without torchrun: start N ranks of this script (one process per
    GPU, RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT set as torchrun
    would), wait for all of them and return the worst exit code.  Rank 0 prints
    the JSON line on the inherited stdout."""
    port = _free_port()
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus), LOCAL_WORLD_SIZE=str(args.gpus),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    codes = [p.wait() for p in procs]
    return max(codes, key=abs)


def init_ranks(args, world: int, local: int, backend: str):
    """One process group over the ranks (NCCL over NVLink for GPUs, gloo for the
    CPU dry run), with NCCL's communicator lines on stderr; returns (barrier,
    max_over_ranks).  max_over_ranks all-reduces a float64 with MAX (device
    tensors under NCCL): every timing in the line is the slowest rank's."""
    import torch
    import torch.distributed as dist
    if world > 1:
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        kw = {"device_id": torch.device("cuda", local)} if backend == "nccl" else {}
        dist.init_process_group(backend, **kw)
    dev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    return barrier, max_over_ranks


CONFIG4_BLOCKS = 8  # config 4 = 8 blocks of 8192 traces x 1024 requests (one N=8 rank's shard each)


def config4_blocks(rank: int, world: int) -> range:
    """This rank's contiguous blocks of config 4 (strong scaling: the 2^26-request
    job is fixed, rank r of N takes blocks [8r/N, 8(r+1)/N))."""
    if CONFIG4_BLOCKS % world:
        raise ValueError("config 4 needs a world size dividing 8")
    from paper_2309_06619_b200 import dist as rdist
    return rdist.shard(rank, world, CONFIG4_BLOCKS)


def dry_run(args):
    """CPU plumbing check (tests): the same rank discovery, process group, config-4
    block sharding, int64 SUM all-reduce (paper_2309_06619_b200.dist, as the GPU
    legs use it) and MAX-over-ranks timing as the native arm, on gloo; each rank's
    "statistics" are synthetic integers derived from its block ids (no kernels,
    no method arithmetic).  Prints the rank-0 JSON line, marked dry_run."""
    import torch
    from paper_2309_06619_b200 import dist as rdist
    rank, world, local = dist_env()
    barrier, max_over_ranks = init_ranks(args, world, local, "gloo")
    t0 = time.perf_counter()
    mine = list(config4_blocks(rank, world))
    sums = torch.zeros((4, 3), dtype=torch.int64)
    for b in mine:  # per-LM rows (sum_resp_us, n, misses) of a stand-in block
        for f in range(4):
            sums[f] += torch.tensor([1000 * (b + 1) + f, 8192 * 1024 // 4, b], dtype=torch.int64)
    rdist.allreduce_sums(sums)
    covered = torch.zeros(CONFIG4_BLOCKS, dtype=torch.int64)
    covered[mine] = 1
    rdist.allreduce_sums(covered)
    barrier()
    ms = max_over_ranks((time.perf_counter() - t0) * 1e3 + rank)  # + rank: MAX must pick the last rank
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
                          "higher_is_better": True, "scaling": "strong", "backend": "gloo",
                          "config4_blocks_covered": covered.tolist(), "sums": sums.tolist(),
                          "max_ms_includes_rank": world - 1}), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock / throttle-reason sampling during the timed region: NVML
    (nvidia_ml_py) every 2 ms, falling back to nvidia-smi every 200 ms."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self._stop.is_set():
            self.rows.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx,
                              pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            self._stop.wait(0.002)
        pynvml.nvmlShutdown()

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        bits = [0x8, 0x40, 0x20, 0x4]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    r = [x.strip() for x in line.split(",")]
                    m = sum(b for b, v in zip(bits, r[2:]) if v == "Active")
                    self.rows.append((float(r[0]), float(r[1]), m))
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        try:
            self._run_nvml()
        except Exception:
            self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({k for r in self.rows for k, b in self.REASONS.items() if int(r[2]) & b})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ native arm
def native(args):
    import torch
    import torch.distributed as dist

    import paper_2309_06619_b200 as rt
    from rtgen import configs

    rank, world, local = dist_env()
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world} (run without torchrun to self-spawn the ranks)")
    barrier, max_over_ranks = init_ranks(args, world, local, "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)

    # ---------------- inputs (config 2 queue, this rank's gid range)
    d2 = configs.config2(n=args.n, gid0=rank * args.n)
    prof = d2["profile"]
    reg = d2["regressor"]
    ctx = rt.Context(d2["lexicon"], local)
    h_bytes = torch.from_numpy(d2["data"]).pin_memory()
    h_off = torch.from_numpy(d2["offsets"].view(np.int32)).pin_memory()
    data = h_bytes.to(dev)
    off = h_off.to(dev)
    n = args.n
    total_bytes = int(d2["offsets"][-1])
    seg = np.asarray([0, n], np.uint32)
    outs = {"u": torch.empty(n, dtype=torch.float32, device=dev), "key": torch.empty(n, dtype=torch.int64, device=dev)}
    souts = {"perm": torch.empty(n, dtype=torch.int32, device=dev), "batch_of": torch.empty(n, dtype=torch.int32, device=dev),
             "slot_of": torch.empty(n, dtype=torch.uint8, device=dev), "core_of": torch.empty(n, dtype=torch.uint8, device=dev),
             "seg_batch_off": torch.empty(2, dtype=torch.int32, device=dev)}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        ctx.score_key(data, off, reg, prof, want_D=False, out=outs)
        ev_mid.record(stream)
        ctx.schedule(outs["key"], outs["u"], seg, prof, out=souts)

    ev_a = torch.cuda.Event(enable_timing=True)
    ev_mid = torch.cuda.Event(enable_timing=True)
    ev_b = torch.cuda.Event(enable_timing=True)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    t_step, t_score = [], []
    for _ in range(args.steps):
        flush.zero_()
        ev_a.record(stream)
        step()
        ev_b.record(stream)
        ev_b.synchronize()
        t_step.append(ev_a.elapsed_time(ev_b))
        t_score.append(ev_a.elapsed_time(ev_mid))
    torch.cuda.synchronize()
    barrier()
    sum_ms = max_over_ranks(sum(t_step))  # one batch at a time, L2 flushed between steps
    score_ms = sum(t_score) / len(t_score)

    # ---------------- pipelined throughput: `depth` batches in flight (one context,
    # stream and distinct 2^20-request input each -> depth x ~100 MB > L2, no flush
    # needed).  Batch k's serial CPU-class chain (one SM) overlaps the following
    # batches' scoring and GPU-class consolidation; every batch still runs the
    # whole hot path.
    depth = max(1, args.depth)
    extra = [configs.config2(n=args.n, gid0=(world * (i + 1) + rank) * args.n) for i in range(depth - 1)]
    ctxs = [ctx] + [rt.Context(d["lexicon"], local) for d in extra]
    h_bytes2 = [h_bytes] + [torch.from_numpy(d["data"]).pin_memory() for d in extra]
    h_off2 = [h_off] + [torch.from_numpy(d["offsets"].view(np.int32)).pin_memory() for d in extra]
    data2 = [data] + [h.to(dev) for h in h_bytes2[1:]]
    off2 = [off] + [h.to(dev) for h in h_off2[1:]]
    streams = [torch.cuda.Stream(dev) for _ in range(depth)]
    outs2 = [outs] + [{k: torch.empty_like(v) for k, v in outs.items()} for _ in extra]
    souts2 = [souts] + [{k: torch.empty_like(v) for k, v in souts.items()} for _ in extra]
    h_res = [{k: torch.empty(n, dtype=dt).pin_memory() for k, dt in (("batch_of", torch.int32), ("slot_of", torch.uint8),
                                                                          ("core_of", torch.uint8))} for _ in range(depth)]

    # scoring of every batch on one stream (in batch order) and each batch's
    # schedule on its slot's stream: the persistent scoring kernels never run two
    # at a time, so they never take the SMs the slots' one-SM list-scheduling
    # chains run on; slot buffers are reused only after the slot's schedule
    score_stream = torch.cuda.Stream(dev)
    ev_scored = [torch.cuda.Event() for _ in range(depth)]
    ev_sched = [torch.cuda.Event() for _ in range(depth)]
    split_streams = os.environ.get("RTLM_SCORE_STREAM", "1") == "1" and not args.graphs

    def pstep(k, e2e=False):
        sl = k % depth
        if e2e or not split_streams:
            with torch.cuda.stream(streams[sl]):
                if e2e:  # the C ABI's host-buffer entry: H2D copies, score+key+schedule, D2H of the assignment
                    ctxs[sl].score_schedule_host(h_bytes2[sl], h_off2[sl], reg, prof, h_res[sl])
                    return
                ctxs[sl].score_key(data2[sl], off2[sl], reg, prof, want_D=False, out=outs2[sl])
                ctxs[sl].schedule(outs2[sl]["key"], outs2[sl]["u"], seg, prof, out=souts2[sl])
            return
        with torch.cuda.stream(score_stream):
            score_stream.wait_event(ev_sched[sl])  # the slot's previous schedule has read u / key
            ctxs[sl].score_key(data2[sl], off2[sl], reg, prof, want_D=False, out=outs2[sl])
            ev_scored[sl].record(score_stream)
        with torch.cuda.stream(streams[sl]):
            streams[sl].wait_event(ev_scored[sl])
            ctxs[sl].schedule(outs2[sl]["key"], outs2[sl]["u"], seg, prof, out=souts2[sl])
            ev_sched[sl].record(streams[sl])

    # --graphs: one CUDA graph per batch slot holding that slot's whole step
    # (rt_score_key + rt_schedule: ~50 kernels, the CPU-class fork/join and the
    # staged offsets), captured once after the warm-up and replayed per step.
    # Measured equal to call-by-call issue (0.867 vs 0.866 ms per step): the
    # step is device-bound, the host only waits on the GPU's progress.
    graphs = [None] * depth
    graph_launches = [0] * depth

    def capture_graphs():
        for sl in range(depth):
            g = torch.cuda.CUDAGraph()
            l0 = rt.launch_count()
            with torch.cuda.graph(g, stream=streams[sl], capture_error_mode="relaxed"):
                pstep(sl, False)
            graph_launches[sl] = rt.launch_count() - l0
            graphs[sl] = g
        torch.cuda.synchronize()

    def gstep(k):
        sl = k % depth
        with torch.cuda.stream(streams[sl]):
            graphs[sl].replay()

    def timed_pipeline(e2e):
        use_graphs = not e2e and args.graphs
        for k in range(max(args.warmup, depth)):  # every slot runs before its capture
            pstep(k, e2e)
        torch.cuda.synchronize()
        if use_graphs and graphs[0] is None:
            capture_graphs()
            for k in range(depth):
                gstep(k)
            torch.cuda.synchronize()
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for st in streams + [score_stream]:
            st.wait_event(t0)
        for k in range(args.steps):
            if use_graphs:
                gstep(k)
            else:
                pstep(k, e2e)
        for st in streams + [score_stream]:
            stream.wait_stream(st)
        t1.record(stream)
        t1.synchronize()
        return t0.elapsed_time(t1)

    # SM partition: the persistent scoring kernel (one at a time, on the scoring
    # stream) gets ~2/3 of the SMs; the slots' schedules (GPU-class consolidation
    # kernels and the one-SM CPU-class list-scheduling chains) run concurrently on
    # the rest.  Measured with k_score6 and 32 hardware queues
    # (profiles/notes/r02_schedule_pipeline.md), 60 steps, two repetitions:
    # 82 / 88 / 94 / 100 / 108 / 116 scoring CTAs -> depth 6: 0.493 / 0.467 /
    # 0.461 / 0.462 / 0.469 / 0.479, depth 8: 0.493 / 0.465 / 0.460 / 0.454 /
    # 0.462 / 0.472 ms per batch.
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    if split_streams:
        score_ctas = max(1, (nsm * 100 + 74) // 148) if depth > 1 else nsm
    else:
        score_ctas = max(1, nsm - depth) if depth > 1 else nsm
    if os.environ.get("RTLM_SCORE_CTAS"):
        score_ctas = int(os.environ["RTLM_SCORE_CTAS"])
    for c in ctxs:
        c.set_sm_limit(score_ctas)
    launches_p0 = rt.launch_count()
    with ClockSampler(local) as clk:
        pipe_ms = max_over_ranks(timed_pipeline(False))
    launches = rt.launch_count() - launches_p0
    if graphs[0] is not None:  # kernels replayed from the graphs (the counter saw the captures only)
        launches = sum(graph_launches[k % depth] for k in range(args.steps))
    clocks = clk.summary()
    e2e_ms = max_over_ranks(timed_pipeline(True))
    for c in ctxs:
        c.set_sm_limit(0)
    value = world * n * args.steps / (pipe_ms / 1e3) / 1e6
    e2e_value = world * n * args.steps / (e2e_ms / 1e3) / 1e6
    mean_bytes = (total_bytes + sum(int(d["offsets"][-1]) for d in extra)) // depth

    # ---------------- roofline of the scoring kernel (k_score: the HBM-bound pass)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak_gbs = float(peaks.get("hbm_gbs", 6650.0))
    alg_bytes = total_bytes + 4 * (n + 1) + 12 * n  # text + offsets + u (4 B) + key (8 B)
    traffic, traffic_src, ncu_note = None, None, None
    try:  # DRAM bytes of one k_score launch from the committed `ncu --set full` capture
        tj = json.load(open(os.path.join(ROOT, "profiles", "k_score_traffic.json")))
        traffic, traffic_src = tj["traffic_bytes"], tj.get("source")
        ncu_note = {k: tj[k] for k in ("issue_slots_busy_pct", "warp_instructions", "note") if k in tj}
    except Exception:
        pass
    achieved = alg_bytes / (score_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": "k_score (rt_score_key)", "achieved": round(achieved, 1),
                "peak": peak_gbs, "unit": "GB/s", "frac": round(achieved / peak_gbs, 4), "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650 GB/s",
                "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": round(score_ms, 5),
                "step_share": round(score_ms / (sum(t_step) / len(t_step)), 4), "ncu": ncu_note}

    # the kernel's binding resource is instruction issue (ncu: ~80 % of issue slots
    # busy at < 4 % of HBM): its issue roofline from the committed ncu instruction
    # count and the live launch time; peak = 148 SMs x 4 schedulers x 1 warp
    # instruction per cycle at the SM clock sampled under load
    if ncu_note and ncu_note.get("warp_instructions"):
        props = torch.cuda.get_device_properties(dev)
        mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
        peak_gips = props.multi_processor_count * 4 * mhz * 1e6 / 1e9
        got_gips = ncu_note["warp_instructions"] / (score_ms / 1e3) / 1e9
        roofline["issue"] = {"bound": "issue", "achieved": round(got_gips, 1), "peak": round(peak_gips, 1),
                             "unit": "G warp-inst/s", "frac": round(got_gips / peak_gips, 4),
                             "warp_instructions_per_launch": ncu_note["warp_instructions"],
                             "peak_source": f"{props.multi_processor_count} SMs x 4 schedulers x {mhz:.0f} MHz"}

    # ---------------- MLP leg (NEXT-1): rt_predict_mlp on config 2's features
    mlp = None
    if not args.no_mlp:
        mlp = mlp_leg(args, rt, ctx, data, off, n, dev, stream, world, barrier, max_over_ranks, flush, peaks)

    # ---------------- offline-profiling leg (NEXT-2): fit + quantile over config 2
    offline = None
    if not args.no_mlp:
        offline = offline_leg(args, ctx, data, off, n, d2, dev, stream, world, max_over_ranks)

    # ---------------- malicious sweep (NEXT-3)
    malicious = None
    if args.sweeps:
        malicious = malicious_leg(args, ctx, configs, dev, rank, max_over_ranks)

    # ---------------- traces leg (config 3 per GPU)
    traces = None
    if not args.no_traces:
        traces = traces_leg(args, rt, ctx, configs, dev, stream, rank, world, barrier, max_over_ranks, flush)

    # ---------------- config 5 sweep (weak: the whole grid over each rank's own traces)
    sweep5 = None
    if not args.no_config5:
        sweep5 = config5_leg(args, ctx, configs, dev, stream, rank, world, barrier, max_over_ranks)

    # ---------------- config 4 (strong: 2^26 requests split over the ranks)
    cfg4 = None
    if not args.no_config4:
        cfg4 = config4_leg(args, ctx, configs, dev, stream, rank, world, barrier, max_over_ranks, flush,
                           lambda: rt.Context(d2["lexicon"], local))

    # ---------------- cpu baseline (oracle, rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_requests_timing(d2, n, reps=4)
        if traces is not None:
            try:
                traces["cpu_baseline"] = oracle_traces_timing(args.per_trace)
            except Exception as e:  # reported, never fatal for the bench line
                traces["cpu_baseline"] = {"error": repr(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(pipe_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8+f32", "data": "synthetic",
            "config": {"workload": "config2: one 2^20-request queue per GPU (DialoGPT profile, all r=0), "
                                   "score+key+schedule", "requests_per_gpu": n, "bytes_per_gpu": total_bytes,
                       "pipeline": f"{depth} batches in flight ({depth} contexts / streams), cycling {depth} distinct inputs, "
                                   f"scoring on {score_ctas} CTAs"
                                   + ("; scoring of every batch on one stream, each batch's schedule on its slot's "
                                      "stream (event-ordered)" if split_streams else "")
                                   + ("; each slot's step replayed from one CUDA graph" if args.graphs else "")
                                   + f"; CUDA_DEVICE_MAX_CONNECTIONS={os.environ.get('CUDA_DEVICE_MAX_CONNECTIONS')}",
                       "l2": f"pipelined: {depth} distinct inputs of ~100 MB each (> 126 MB L2) in turn; "
                             "latency leg: 256 MB buffer written between steps",
                       "parallelism": f"replicas{world}",
                       "lexicon_sha256": hashlib.sha256(d2["lexicon"]).hexdigest(),
                       "seed": "rtgen ROOT_SEED + 2 (counter-based; gid range rank * n ..)"},
            "latency": {"ms_per_step": round(sum_ms / args.steps, 4), "score_key_ms": round(score_ms, 4),
                        "schedule_ms": round(sum(t_step) / len(t_step) - score_ms, 4),
                        "note": "one batch at a time, L2 flushed between steps"},
            "e2e": {"value": round(e2e_value, 3), "unit": UNIT,
                    "h2d_bytes_per_step": mean_bytes + 4 * (n + 1),
                    "d2h_bytes_per_step": 6 * n, "ms_per_step": round(e2e_ms / args.steps, 4),
                    "path": "rt_score_schedule_host (C ABI): pinned host text + offsets -> H2D, score+key+schedule, "
                            "D2H of batch/slot/core; one context and stream per in-flight batch"},
            "gpu_launches": int(launches),
            "ranks": {"world": world, "backend": "nccl" if world > 1 else None,
                      "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if world > 1 else None,
                      "launch": "torchrun" if os.environ.get("TORCHELASTIC_RUN_ID") else
                                ("self-spawned (bench.py --gpus N)" if world > 1 else "single process")},
            "roofline": roofline,
            "clocks": clocks,
        }
        if traces is not None:
            line["traces"] = traces
        if mlp is not None:
            line["mlp"] = mlp
        if offline is not None:
            line["offline"] = offline
        if malicious is not None:
            line["malicious"] = malicious
        if sweep5 is not None:
            line["config5"] = sweep5
        if cfg4 is not None:
            line["config4"] = cfg4
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def mlp_leg(args, rt, ctx, data, off, n, dev, stream, world, barrier, max_over_ranks, flush, peaks):
    """NEXT-1: u = m_theta(feat) for the config-2 queue (features from rt_score),
    random-init weights (no trained model exists here; the cost does not depend
    on the values), in three precisions: fp32 (default; CUDA-core binary32 FMA
    chains, k_mlp_f32), tf32x3 (fp32-accurate on tcgen05: three TF32 products
    per multiply, k_mlp_tf32) and bf16 (opt-in; tcgen05, k_mlp).  Algorithmic
    2 * 80 700 FLOP per request.  Rooflines: fp32 against the CUDA-core FMA
    peak (148 SMs x 128 FP32 lanes x 2 FLOP x the SM clock, derived: the
    profiling guide and MEASURED_PEAKS.json give no fp32 number); tf32x3
    against the emulated-fp32 peak = the tf32 peak / 3, the tf32 peak being
    MEASURED_PEAKS.json bf16_tflops x 1.1 / 2.25 (the guide's nominal tf32 :
    bf16 ratio); bf16 against MEASURED_PEAKS.json bf16_tflops."""
    import torch
    import rtgen
    feat = ctx.score(data, off)
    ws, bs = rtgen.mlp_weights(12345)
    ctx.set_mlp(ws, bs)
    u = torch.empty(n, dtype=torch.float32, device=dev)
    flops = 2 * (6 * 100 + 100 * 200 + 200 * 200 + 200 * 100 + 100) * n
    props = torch.cuda.get_device_properties(dev)
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    out = {"metric": "M requests/s (u = m_theta(feat), MLP 6-100-200-200-100-1)", "unit": "Mreq/s",
           "alg_flops_per_launch": flops}
    for prec in ("fp32", "tf32x3", "bf16"):
        ctx.set_mlp_precision(prec)
        for _ in range(args.warmup):
            ctx.predict_mlp(feat, u)
        torch.cuda.synchronize()
        barrier()
        ev_a = torch.cuda.Event(enable_timing=True)
        ev_b = torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(max(3, args.steps // 4) if prec == "fp32" else args.steps):
            flush.zero_()
            ev_a.record(stream)
            ctx.predict_mlp(feat, u)
            ev_b.record(stream)
            ev_b.synchronize()
            ts.append(ev_a.elapsed_time(ev_b))
        ms = max_over_ranks(sum(ts)) / len(ts)
        achieved = flops / (ms / 1e3) / 1e12
        if prec == "fp32":
            peak = props.multi_processor_count * 128 * 2 * mhz * 1e6 / 1e12
            roof = {"bound": "alu", "kernel": "k_mlp_f32", "achieved": round(achieved, 2), "peak": round(peak, 2),
                    "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": None,
                    "peak_source": f"derived: {props.multi_processor_count} SMs x 128 FP32 FMA/clk x 2 x {mhz:.0f} MHz"}
            dtype = "fp32 CUDA cores (binary32 FMA chains in index order)"
        elif prec == "tf32x3":
            bf16 = float(peaks.get("bf16_tflops", 2250.0))
            peak = bf16 * 1.1 / 2.25 / 3
            roof = {"bound": "tensor", "kernel": "k_mlp_tf32", "achieved": round(achieved, 1), "peak": round(peak, 1),
                    "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": None,
                    "peak_source": ("MEASURED_PEAKS.json bf16_tflops" if "bf16_tflops" in peaks else "nominal bf16")
                    + " x 1.1/2.25 (tf32, guide ratio) / 3 (three tf32 products per fp32 multiply)"}
            dtype = "fp32-accurate: 3xTF32 on tcgen05 (hi/lo split operands), fp32 accumulate in TMEM"
        else:
            peak = float(peaks.get("bf16_tflops", 2250.0))
            roof = {"bound": "tensor", "kernel": "k_mlp", "achieved": round(achieved, 1), "peak": peak,
                    "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": None,
                    "peak_source": "MEASURED_PEAKS.json bf16_tflops" if "bf16_tflops" in peaks else "nominal"}
            dtype = "bf16 tensor cores (tcgen05), fp32 accumulate; layers 1/5 fp32"
        out[prec] = {"value": round(world * n / (ms / 1e3) / 1e6, 2), "ms_per_step": round(ms, 4), "dtype": dtype,
                     "roofline": roof}
    ctx.set_mlp_precision("fp32")
    out["value"] = out["fp32"]["value"]  # the default precision
    return out


def offline_leg(args, ctx, data, off, n, d2, dev, stream, world, max_over_ranks):
    """NEXT-2: weighted-rule fit (normal equations, fp64) over the 2^20 config-2
    records (features from rt_score, targets = true lengths) and the nearest-rank
    0.9-quantile + max of u (tau, u_max).  Algorithmic bytes: 20 B/record (fit),
    the sort's 5 passes x 24 B/record for the quantile."""
    import torch
    import rtgen
    feat = ctx.score(data, off)
    y = torch.from_numpy(d2["true_len"].astype(np.float32)).to(dev)
    u = torch.rand(n, device=dev) * 100
    ev_a = torch.cuda.Event(enable_timing=True)
    ev_b = torch.cuda.Event(enable_timing=True)

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        ev_a.record(stream)
        for _ in range(args.steps):
            fn()
        ev_b.record(stream)
        ev_b.synchronize()
        return max_over_ranks(ev_a.elapsed_time(ev_b)) / args.steps

    fit_ms = timed(lambda: ctx.fit_rule(feat, y))
    q_ms = timed(lambda: ctx.quantile(u, 0.9))
    # MLP training (rt_train_mlp, Adam, lr 1e-4 as P:620): one epoch over the
    # 65 536-record training sample of the calibration in batches of
    # 256; the paper trains 100 epochs at ~3 s per epoch on its board
    ntr = min(n, 65536)
    ws, bs = rtgen.mlp_weights(2024)
    ctx.set_mlp(ws, bs)
    ft, yt = feat[:ntr], y[:ntr]
    t0 = time.perf_counter()
    ctx.train_mlp(ft, yt, 1, 256, 1e-4, 7)
    ep_s = time.perf_counter() - t0
    flops = 3 * 2 * (6 * 100 + 100 * 200 + 200 * 200 + 200 * 100 + 100) * ntr  # forward + 2 backward GEMMs
    return {"fit_ms": round(fit_ms, 4), "fit_Mrec_per_s": round(world * n / (fit_ms / 1e3) / 1e6, 1),
            "fit_GBps": round(20 * n / (fit_ms / 1e3) / 1e9, 1),
            "quantile_ms": round(q_ms, 4), "quantile_Mrec_per_s": round(world * n / (q_ms / 1e3) / 1e6, 1),
            "records_per_gpu": n,
            "train_mlp": {"epoch_s": round(ep_s, 4), "records": ntr, "batch": 256, "lr": 1e-4,
                          "records_per_s": round(ntr / ep_s, 1), "TFLOPs": round(flops / ep_s / 1e12, 3),
                          "note": "wall clock of one rt_train_mlp epoch (it synchronizes): 256 Adam steps of ~22 "
                                  "launches each, fp32 CUDA-core GEMMs"}}


def run_traces_once(ctx, d, dev, profile_overrides=None):
    """Score (per LM group) + replay one traces() workload on the device; returns
    (total µs of response, tasks, misses, device ms).  Groups must be contiguous."""
    import torch
    n = len(d["arrival_us"])
    off_np = d["offsets"]
    arr = torch.from_numpy(d["arrival_us"]).to(dev)
    tl = torch.from_numpy(d["true_len"].view(np.int16)).to(dev)
    tp = torch.from_numpy(d["trace_prof"].view(np.int16)).to(dev)
    profs = [dict(p, **(profile_overrides or {})) for p in d["profiles"]]
    u = torch.empty(n, dtype=torch.float32, device=dev)
    key = torch.empty(n, dtype=torch.int64, device=dev)
    D = torch.empty(n, dtype=torch.int32, device=dev)
    groups = _lm_groups(d, dev)  # raises on non-contiguous LM ranges
    ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_a.record()
    for f, r0, r1, gd, so in groups:
        ctx.score_key(gd, so, d["regressors"][f], profs[f], arrival=arr[r0:r1],
                      out={"u": u[r0:r1], "key": key[r0:r1], "D": D[r0:r1]})
    stats, _ = ctx.simulate(arr, tl, u, key, D, d["trace_off"], profs, tp)
    ev_b.record()
    ev_b.synchronize()
    import paper_2309_06619_b200 as rt
    st = rt.decode_stats(stats)
    return int(st["sum_resp_us"].sum()), int(st["n"].sum()), int(st["misses"].sum()), ev_a.elapsed_time(ev_b)


def malicious_leg(args, ctx, configs, dev, rank, max_over_ranks):
    """NEXT-3: malicious-task ratio sweep 0..100 % in steps of 10 %:
    crafted suffix + x3 true length on a seeded fraction of the requests; UP+C+O
    (the profiles as calibrated) against FIFO without consolidation / offloading.
    128 traces x 1000 requests per point, at two operating points: the paper's
    ramp with tight deadlines (x1/tight: every task is overdue on arrival, so
    the policies can only differ in response time) and an 8x faster ramp with
    loose deadlines (x8/loose, config 5's knee: queues form, ready sets hold
    many tasks, and the policies' orders matter).  Statistics, not gated."""
    nt = 128
    first = 10000 + rank * nt
    ratios = [round(0.1 * i, 1) for i in range(11)]
    out = {"ratios": ratios, "traces_per_point": nt}
    dev_ms = 0.0
    for op, mult, tight in (("x1/tight", 1.0, 1), ("x8/loose", 8.0, 2)):
        base = configs.traces(3, range(first, first + nt), 1000, lambda t: ((t - first) * 4) // nt,
                              beta0=10.0 * mult, step=mult, beta_max=150.0 * mult)
        res = {"mean_response_s": {"UP+C+O": [], "FIFO": []}, "miss_ratio": {"UP+C+O": [], "FIFO": []}}
        for r in ratios:
            d = configs.with_malicious(base, r)
            for name, ov in (("UP+C+O", {"tightness": tight}),
                             ("FIFO", {"policy": "FIFO", "consolidate": 0, "offload": 0, "tightness": tight})):
                resp, cnt, miss, ms = run_traces_once(ctx, d, dev, ov)
                dev_ms += ms
                res["mean_response_s"][name].append(round(resp / max(cnt, 1) / 1e6, 4))
                res["miss_ratio"][name].append(round(miss / max(cnt, 1), 4))
        out[op] = res
    # periodic release: each task released at the previous task's
    # deadline, tight / loose; deadlines from the GPU path (rt_score_key)
    out["periodic"] = periodic_leg(ctx, configs.traces(3, range(12000 + rank * nt, 12000 + (rank + 1) * nt), 1000,
                                                       lambda t: ((t - 12000 - rank * nt) * 4) // nt), dev)
    # the variance subsets are single-LM DialoGPT traces: queues form only above
    # ~x32 (a C = 11 batch of ~1.5 s serves ~400 tasks per minute)
    out["variance"] = {op: variance_leg(ctx, rank, dev, mult, tight) for op, mult, tight in
                       (("x1/tight", 1.0, 1), ("x32/loose", 32.0, 2))}
    out["device_ms_total"] = round(max_over_ranks(dev_ms), 3)
    out["traces_per_s"] = round(nt * len(ratios) * 4 / (out["device_ms_total"] / 1e3), 1)
    out["note"] = ("statistics of the synthetic workload, not gated; x1/tight: config 3's tight deadlines make "
                   "every task overdue on arrival; x8/loose: queues form, so the orders of the policies differ")
    return out


def variance_leg(ctx, rank, dev, mult=1.0, tight=1):
    """NEXT-3 variance subsets: a DialoGPT pool of 64 traces x 1000
    requests scored on the GPU; 20 000 tasks each with small / medium / large
    spread of u (configs.variance_subsets), packed into 20 Poisson traces of
    1000; mean response time for FIFO, LUF, MUF (no consolidation / offload)
    and UP+C+O.  Statistics, not gated."""
    import torch
    import rtgen
    from rtgen import configs
    import paper_2309_06619_b200 as rt
    nt_pool, per, size = 64, 1000, 20000
    first = 14000 + rank * nt_pool
    pool = configs.traces(3, range(first, first + nt_pool), per, lambda t: 0)
    n = len(pool["true_len"])
    feat = torch.empty((n, 8), dtype=torch.int16, device=dev)
    u = torch.empty(n, dtype=torch.float32, device=dev)
    tmpk = torch.empty(n, dtype=torch.int64, device=dev)
    for f, r0, r1, gd, so in _lm_groups(pool, dev):
        ctx.score_key(gd, so, pool["regressors"][f], pool["profiles"][f], want_feat=True, want_D=False,
                      out={"u": u[r0:r1], "key": tmpk[r0:r1], "feat": feat[r0:r1]})
    subs = configs.variance_subsets(u.cpu().numpy(), size)
    nt = size // per
    toff = (np.arange(nt + 1) * per).astype(np.uint32)
    arr = torch.from_numpy(np.concatenate([rtgen.arrivals(rtgen.ROOT_SEED + 3, 900000 + first + t, per, 10.0 * mult,
                                                          mult, 150.0 * mult) for t in range(nt)])).to(dev)
    tp = torch.zeros(nt, dtype=torch.int16, device=dev)
    tl_all = torch.from_numpy(pool["true_len"].view(np.int16)).to(dev)
    pols = {"FIFO": {"policy": "FIFO", "consolidate": 0, "offload": 0},
            "LUF": {"policy": "LUF", "consolidate": 0, "offload": 0},
            "MUF": {"policy": "MUF", "consolidate": 0, "offload": 0}, "UP+C+O": {}}
    res = {}
    for which, idx in subs.items():
        ix = torch.from_numpy(idx.astype(np.int64)).to(dev)
        fs, us, tl = feat[ix].contiguous(), u[ix].contiguous(), tl_all[ix].contiguous()
        row = {"u_std": round(float(us.std().item()), 3)}
        for name, ov in pols.items():
            prof = dict(pool["profiles"][0], tightness=tight, **ov)
            key, D = ctx.key(us, prof, feat=fs, arrival=arr)
            stats, _ = ctx.simulate(arr, tl, us, key, D, toff, [prof], tp)
            st = rt.decode_stats(stats)
            row[name] = round(float(st["sum_resp_us"].sum()) / max(1, int(st["n"].sum())) / 1e6, 4)
        res[which] = row
    return {"mean_response_s": res, "tasks_per_subset": size, "rate_multiplier": mult, "tightness": tight}


def periodic_leg(ctx, base, dev):
    """Miss ratio under periodic release for UP+C+O, EDF, LUF, MUF,
    tight and loose deadlines; arrivals r_{i+1} = r_i + D_i from the device-computed
    deadlines (statistics, not gated)."""
    import torch
    from rtgen import configs
    import paper_2309_06619_b200 as rt
    n = len(base["arrival_us"])
    feat = torch.empty((n, 8), dtype=torch.int16, device=dev)
    u = torch.empty(n, dtype=torch.float32, device=dev)
    tmpk = torch.empty(n, dtype=torch.int64, device=dev)
    groups = _lm_groups(base, dev)
    for f, r0, r1, gd, so in groups:
        ctx.score_key(gd, so, base["regressors"][f], base["profiles"][f], want_feat=True, want_D=False,
                      out={"u": u[r0:r1], "key": tmpk[r0:r1], "feat": feat[r0:r1]})
    tl = torch.from_numpy(base["true_len"].view(np.int16)).to(dev)
    tp = torch.from_numpy(base["trace_prof"].view(np.int16)).to(dev)
    pols = {"UP+C+O": {}, "EDF": {"policy": "EDF", "consolidate": 0, "offload": 0},
            "LUF": {"policy": "LUF", "consolidate": 0, "offload": 0},
            "MUF": {"policy": "MUF", "consolidate": 0, "offload": 0}}
    res = {}
    for tight in (1, 2):
        for name, ov in pols.items():
            profs = [dict(p, tightness=tight, **ov) for p in base["profiles"]]
            D = torch.empty(n, dtype=torch.int32, device=dev)
            key = torch.empty(n, dtype=torch.int64, device=dev)
            for f, r0, r1, gd, so in groups:
                ctx.key(u[r0:r1], profs[f], feat=feat[r0:r1], key=key[r0:r1], D_out=D[r0:r1])
            arr_np = configs.periodic_arrivals(base["trace_off"], D.cpu().numpy().view(np.uint32))
            arr = torch.from_numpy(arr_np).to(dev)
            for f, r0, r1, gd, so in groups:  # EDF keys depend on the release times
                ctx.key(u[r0:r1], profs[f], feat=feat[r0:r1], arrival=arr[r0:r1], key=key[r0:r1], D_out=D[r0:r1])
            stats, _ = ctx.simulate(arr, tl, u, key, D, base["trace_off"], profs, tp)
            st = rt.decode_stats(stats)
            res[f"{name}/{'tight' if tight == 1 else 'loose'}"] = round(float(st["misses"].sum()) / max(1, int(st["n"].sum())), 4)
    return {"miss_ratio": res, "traces": len(base["trace_off"]) - 1}


def traces_leg(args, rt, ctx, configs, dev, stream, rank, world, barrier, max_over_ranks, flush):
    import torch
    from paper_2309_06619_b200 import dist as rdist
    nt = args.traces
    per_lm = max(1, nt // 4)
    first = rank * nt
    d = configs.traces(3, range(first, first + nt), args.per_trace, lambda t: ((t % nt) // per_lm) % 4)
    n = len(d["arrival_us"])
    data = torch.from_numpy(d["data"]).to(dev)
    off_np = d["offsets"]
    off = torch.from_numpy(off_np.view(np.int32)).to(dev)
    arr = torch.from_numpy(d["arrival_us"]).to(dev)
    tl = torch.from_numpy(d["true_len"].view(np.int16)).to(dev)
    tp = torch.from_numpy(d["trace_prof"].view(np.int16)).to(dev)
    u = torch.empty(n, dtype=torch.float32, device=dev)
    key = torch.empty(n, dtype=torch.int64, device=dev)
    D = torch.empty(n, dtype=torch.int32, device=dev)
    stats = torch.empty((nt, 2), dtype=torch.int64, device=dev)
    sums = torch.zeros((4, 3), dtype=torch.int64, device=dev)
    # contiguous request ranges per LM (traces t*per_lm .. ) -> one score_key launch per LM
    groups = []
    for f in range(4):
        sel = np.nonzero(d["trace_prof"] == f)[0]
        if len(sel) == 0:
            continue
        t0, t1 = int(sel[0]), int(sel[-1]) + 1
        r0, r1 = int(d["trace_off"][t0]), int(d["trace_off"][t1])
        sub_off = torch.from_numpy((off_np[r0:r1 + 1] - off_np[r0]).astype(np.uint32).view(np.int32)).to(dev)
        b0 = int(off_np[r0])
        align = b0 & ~15
        groups.append((f, r0, r1, b0, align, sub_off))
    # score_key requires 16-byte-aligned text: re-base each group's bytes into its own aligned buffer
    gdata = [data[b0:int(off_np[r1])].clone() for (f, r0, r1, b0, align, so) in groups]
    grp_of = torch.from_numpy(d["trace_prof"].view(np.int16)).to(dev)

    def step():
        for (f, r0, r1, b0, align, so), gd in zip(groups, gdata):
            ctx.score_key(gd, so, d["regressors"][f], d["profiles"][f], arrival=arr[r0:r1],
                          out={"u": u[r0:r1], "key": key[r0:r1], "D": D[r0:r1]})
        ctx.simulate(arr, tl, u, key, D, d["trace_off"], d["profiles"], tp, stats=stats)
        sums.zero_()
        ctx.reduce_stats(stats, grp_of, 4, sums=sums)
        rdist.allreduce_sums(sums)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    ev_a = torch.cuda.Event(enable_timing=True)
    ev_b = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(args.steps):
        flush.zero_()
        ev_a.record(stream)
        step()
        ev_b.record(stream)
        ev_b.synchronize()
        ts.append(ev_a.elapsed_time(ev_b))
    tsum = max_over_ranks(sum(ts))
    # NEXT-4: per-trace max / p95 response and makespan from the end times (one extra replay with end times)
    _, end = ctx.simulate(arr, tl, u, key, D, d["trace_off"], d["profiles"], tp, want_end=True)
    ev_a.record(stream)
    rep = ctx.trace_report(arr, end, d["trace_off"])
    ev_b.record(stream)
    util = ctx.trace_utilization(tl, key, end, d["trace_off"], d["profiles"], tp)
    ev_c = torch.cuda.Event(enable_timing=True)
    ev_c.record(stream)
    ev_c.synchronize()
    report_ms = ev_a.elapsed_time(ev_b)
    util_ms = ev_b.elapsed_time(ev_c)
    rep = rep.cpu().numpy()
    util = util.cpu().numpy()
    tprof = d["trace_prof"]
    p95 = [float(np.median(rep[tprof == f, 1])) / 1e6 if (tprof == f).any() else None for f in range(4)]
    cores = np.array([d["profiles"][int(f)]["cores"] for f in tprof], np.float64)
    mk = np.maximum(rep[:, 2], 1).astype(np.float64)
    gfrac = util[:, 0] / mk
    cfrac = util[:, 1] / (mk * np.maximum(cores, 1))
    gutil = [round(float(np.mean(gfrac[tprof == f])), 4) if (tprof == f).any() else None for f in range(4)]
    cutil = [round(float(np.mean(cfrac[tprof == f])), 4) if (tprof == f).any() else None for f in range(4)]
    s = sums.cpu().numpy()
    mean_resp = [float(s[f, 0]) / max(1, s[f, 1]) / 1e6 for f in range(4)]
    miss = [float(s[f, 2]) / max(1, s[f, 1]) for f in range(4)]
    return {"metric": "traces/s", "value": round(world * nt * args.steps / (tsum / 1e3), 1), "unit": "traces/s",
            "requests_per_s": round(world * n * args.steps / (tsum / 1e3), 1),
            "ms_per_step": round(tsum / args.steps, 4),
            "workload": f"config3: {nt} Poisson-ramp traces x {args.per_trace} requests per GPU, 4 LMs, tight, UP+C+O",
            "mean_response_s_per_lm": [round(x, 4) for x in mean_resp], "miss_ratio_per_lm": [round(x, 4) for x in miss],
            "median_p95_response_s_per_lm": [None if x is None else round(x, 4) for x in p95],
            "mean_gpu_util_per_lm": gutil, "mean_cpu_util_per_lm": cutil,
            "trace_report_ms": round(report_ms, 4), "trace_util_ms": round(util_ms, 4)}


def _lm_groups(d, dev):
    """Contiguous per-LM request ranges of a traces() workload: (lm, r0, r1,
    16-byte-aligned copy of the group's text, group-relative offsets)."""
    import torch
    off_np = d["offsets"]
    groups = []
    for f in range(4):
        sel = np.nonzero(d["trace_prof"] == f)[0]
        if len(sel) == 0:
            continue
        t0, t1 = int(sel[0]), int(sel[-1]) + 1
        if t1 - t0 != len(sel):
            raise ValueError("LM groups must be contiguous trace ranges")
        r0, r1 = int(d["trace_off"][t0]), int(d["trace_off"][t1])
        b0, b1 = int(off_np[r0]), int(off_np[r1])
        so = torch.from_numpy((off_np[r0:r1 + 1] - off_np[r0]).astype(np.uint32).view(np.int32)).to(dev)
        groups.append((f, r0, r1, torch.from_numpy(np.ascontiguousarray(d["data"][b0:b1])).to(dev), so))
    return groups


def config5_leg(args, ctx, configs, dev, stream, rank, world, barrier, max_over_ranks):
    """BASELINE configs[4]: the arrival-rate x deadline x ablation sweep
    (SURVEY §8(d) config 5): 154 points (8 rate multipliers x tightness 1/2 x
    FIFO/HPF/LUF/MUF/UP/UP+C/UP+C+O, plus alpha 0-2 and b 1.0-3.0 on UP+C+O),
    each over 64 traces x 1000 requests per LM (256 traces).  Features and u are
    scored once (rt_score_key); a step recomputes every point's keys and
    deadlines (rt_key, one launch per point and LM) and replays the whole grid
    as ONE rt_simulate over 154 x 256 traces (per-trace profile index = point x 4
    + LM), then sums per (point, LM) (rt_reduce_stats) and all-reduces them (a8).
    Weak scaling: every rank runs the grid over its own traces."""
    import torch
    from paper_2309_06619_b200 import dist as rdist
    per_lm = 64
    base = configs.config5_base(20000 + rank * 4 * per_lm, per_lm)
    pts = configs.config5_points()
    npt = len(pts)
    n = len(base["arrival_us"])
    nt = len(base["trace_off"]) - 1
    groups = _lm_groups(base, dev)
    arr_m = {m: torch.from_numpy(configs.config5_arrivals(base, m)).to(dev) for m in configs.CONFIG5_MULTS}
    feat = torch.empty((n, 8), dtype=torch.int16, device=dev)
    u = torch.empty(n, dtype=torch.float32, device=dev)
    tmpk = torch.empty(n, dtype=torch.int64, device=dev)
    for f, r0, r1, gd, so in groups:  # scoring once (features + u per LM regressor)
        ctx.score_key(gd, so, base["regressors"][f], base["profiles"][f], want_feat=True, want_D=False,
                      out={"u": u[r0:r1], "key": tmpk[r0:r1], "feat": feat[r0:r1]})
    # the grid as one trace set: point i's traces are i*nt .. (i+1)*nt - 1
    arr = torch.cat([arr_m[pt["mult"]] for pt in pts])
    tl = torch.from_numpy(base["true_len"].view(np.int16)).to(dev).repeat(npt)
    u_all = u.repeat(npt)
    key = torch.empty(npt * n, dtype=torch.int64, device=dev)
    D = torch.empty(npt * n, dtype=torch.int32, device=dev)
    tprof = torch.from_numpy(np.concatenate([base["trace_prof"].astype(np.int64) + 4 * i for i in range(npt)])
                             .astype(np.uint16).view(np.int16)).to(dev)
    toff = (np.arange(npt * nt + 1, dtype=np.uint64) * int(base["trace_off"][1])).astype(np.uint32)
    profs = [dict(p, **pt["overrides"]) for pt in pts for p in base["profiles"]]
    stats = torch.empty((npt * nt, 2), dtype=torch.int64, device=dev)
    sums = torch.zeros((npt * 4, 3), dtype=torch.int64, device=dev)

    def grid():
        for i in range(npt):
            o = i * n
            for f, r0, r1, gd, so in groups:
                ctx.key(u[r0:r1], profs[4 * i + f], feat=feat[r0:r1], arrival=arr[o + r0:o + r1],
                        key=key[o + r0:o + r1], D_out=D[o + r0:o + r1])
        ctx.simulate(arr, tl, u_all, key, D, toff, profs, tprof, stats=stats)
        sums.zero_()
        ctx.reduce_stats(stats, tprof, npt * 4, sums=sums)
        rdist.allreduce_sums(sums)

    steps = max(1, min(args.steps, 5))
    for _ in range(max(1, min(args.warmup, 3))):
        grid()
    torch.cuda.synchronize()
    barrier()
    ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_a.record(stream)
    for _ in range(steps):
        grid()
    ev_b.record(stream)
    ev_b.synchronize()
    ms = max_over_ranks(ev_a.elapsed_time(ev_b)) / steps
    s = sums.cpu().numpy().reshape(npt, 4, 3).sum(axis=1)  # over LMs
    mean_resp = (s[:, 0] / np.maximum(s[:, 1], 1) / 1e6).round(4)
    miss = (s[:, 2] / np.maximum(s[:, 1], 1)).round(4)
    by_policy = {}
    for tight in (1, 2):
        for name in configs.CONFIG5_POLICIES:
            idx = [i for i, p in enumerate(pts) if p["name"] == f"{name}/t{tight}"]
            by_policy[f"{name}/t{tight}"] = {"mean_response_s": [float(mean_resp[i]) for i in idx],
                                             "miss_ratio": [float(miss[i]) for i in idx]}
    ab = lambda pre, arr_: [float(arr_[i]) for i, p in enumerate(pts) if p["name"].startswith(pre)]
    traces_total = world * npt * nt
    return {"metric": "traces/s", "value": round(traces_total / (ms / 1e3), 1), "unit": "traces/s",
            "requests_per_s": round(traces_total * (n // max(nt, 1)) / (ms / 1e3), 1),
            "ms_per_grid": round(ms, 3), "points": npt, "traces_per_point_per_gpu": nt,
            "workload": "config5: 154 points (rate x0.25..x32 x tightness 1/2 x 7 policies; alpha 0-2 and b 1.0-3.0 "
                        f"on UP+C+O at rate x{configs.CONFIG5_AB_MULT:g}, tightness {configs.CONFIG5_AB_TIGHTNESS}) "
                        "x 64 traces x 1000 requests per LM per GPU; keys recomputed per point, one replay launch",
            "scaling": "weak", "mults": list(configs.CONFIG5_MULTS), "by_policy": by_policy,
            "alpha": {"mean_response_s": ab("alpha=", mean_resp), "miss_ratio": ab("alpha=", miss)},
            "b": {"mean_response_s": ab("b=", mean_resp), "miss_ratio": ab("b=", miss)}}


def config4_leg(args, ctx, configs, dev, stream, rank, world, barrier, max_over_ranks, flush, make_ctx):
    """BASELINE configs[3]: 2^26 requests = 65536 traces x 1024, contiguous trace
    ranges per rank (strong scaling: the job is fixed, each rank takes 1/N of
    it), score_key per LM + replay + stats, one NCCL all-reduce of the per-LM
    int64 sums (a8).  value = 2^26 requests / max-over-ranks step time.
    The rank's blocks (8192 traces each) alternate between two contexts and
    streams, so that one block's scoring (issue-bound, whole SMs) overlaps the
    other's replay (latency-bound one-warp CTAs); the per-LM sums are
    accumulated by both with atomics."""
    import torch
    from paper_2309_06619_b200 import dist as rdist
    t0 = time.time()
    # blocks of 8192 traces (one N=8 rank's shard; u32 text offsets per block)
    blocks = []
    for blk in config4_blocks(rank, world):
        d = configs.config4_shard(blk, CONFIG4_BLOCKS, grouped=True)
        nb, ntb = len(d["arrival_us"]), len(d["trace_off"]) - 1
        blocks.append({"d": d, "groups": _lm_groups(d, dev),
                       "arr": torch.from_numpy(d["arrival_us"]).to(dev),
                       "tl": torch.from_numpy(d["true_len"].view(np.int16)).to(dev),
                       "tp": torch.from_numpy(d["trace_prof"].view(np.int16)).to(dev),
                       "u": torch.empty(nb, dtype=torch.float32, device=dev),
                       "key": torch.empty(nb, dtype=torch.int64, device=dev),
                       "D": torch.empty(nb, dtype=torch.int32, device=dev),
                       "stats": torch.empty((ntb, 2), dtype=torch.int64, device=dev)})
        del d["data"]
    gen_s = time.time() - t0
    n = sum(len(b["d"]["arrival_us"]) for b in blocks)
    nt = sum(len(b["d"]["trace_off"]) - 1 for b in blocks)
    sums = torch.zeros((4, 3), dtype=torch.int64, device=dev)
    nstreams = max(1, int(os.environ.get("RTLM_C4_STREAMS", "2")))
    ctxs = [ctx] + [make_ctx() for _ in range(nstreams - 1)]
    streams = [torch.cuda.Stream(dev) for _ in range(nstreams)]
    # scoring capped at half the SMs so that it leaves room for the other
    # stream's replay: 48.0 ms (one stream) -> 47.4 (two) -> 46.3 / 46.0 (two,
    # scoring on 100 / 74 CTAs) per 2^26 requests
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    c4_ctas = int(os.environ.get("RTLM_C4_SCORE_CTAS", str((nsm + 1) // 2 if nstreams > 1 else 0)))
    for c in ctxs:
        c.set_sm_limit(c4_ctas)
    ev0 = torch.cuda.Event()

    def step():
        sums.zero_()
        ev0.record(stream)
        for i, b in enumerate(blocks):
            c, st = ctxs[i % nstreams], streams[i % nstreams]
            with torch.cuda.stream(st):
                if i < nstreams:
                    st.wait_event(ev0)
                d, u, key, D, arr = b["d"], b["u"], b["key"], b["D"], b["arr"]
                for f, r0, r1, gd, so in b["groups"]:
                    c.score_key(gd, so, d["regressors"][f], d["profiles"][f], arrival=arr[r0:r1],
                                out={"u": u[r0:r1], "key": key[r0:r1], "D": D[r0:r1]})
                c.simulate(arr, b["tl"], u, key, D, d["trace_off"], d["profiles"], b["tp"], stats=b["stats"])
                c.reduce_stats(b["stats"], b["tp"], 4, sums=sums)
        for st in streams:
            stream.wait_stream(st)
        rdist.allreduce_sums(sums)

    steps = max(1, min(args.steps, 5))
    for _ in range(max(1, min(args.warmup, 3))):
        step()
    torch.cuda.synchronize()
    barrier()
    ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(steps):
        flush.zero_()
        ev_a.record(stream)
        step()
        ev_b.record(stream)
        ev_b.synchronize()
        ts.append(ev_a.elapsed_time(ev_b))
    ms = max_over_ranks(sum(ts)) / steps
    for c in ctxs:
        c.set_sm_limit(0)
    s = sums.cpu().numpy()
    total_req = 65536 * 1024
    return {"metric": "M requests scored+scheduled+replayed/s", "value": round(total_req / (ms / 1e3) / 1e6, 2),
            "unit": "Mreq/s", "traces_per_s": round(65536 / (ms / 1e3), 1), "ms_per_step": round(ms, 3),
            "scaling": "strong", "requests_per_gpu": n, "traces_per_gpu": nt, "host_gen_s": round(gen_s, 1),
            "streams": nstreams, "score_ctas": c4_ctas or None,
            "workload": "config4: 65536 Poisson-ramp traces x 1024 requests (2^26) split over the ranks, 4 LMs, "
                        "tight, UP+C+O; one NCCL all-reduce of per-LM int64 sums",
            "mean_response_s_per_lm": [round(float(s[f, 0]) / max(1, s[f, 1]) / 1e6, 4) for f in range(4)],
            "miss_ratio_per_lm": [round(float(s[f, 2]) / max(1, s[f, 1]), 4) for f in range(4)]}


def _oracle_traces_worker(args):
    """One host process of the traces CPU baseline: the oracle (single thread, as
    it stands) scores, keys and replays its own config-3 traces; returns (traces,
    seconds of oracle work)."""
    first, count, per_trace = args
    import oracle
    from rtgen import configs
    per_lm = 1024
    d = configs.traces(3, range(first, first + count), per_trace, lambda t: (t // per_lm) % 4)
    lex = oracle.Lexicon(d["lexicon"])
    t0 = time.time()
    f = oracle.rule_gen(lex, d["data"], d["offsets"])
    n = len(f)
    u = np.zeros(n, np.float32)
    k = np.zeros(n, np.uint64)
    D = np.zeros(n, np.uint32)
    for t in range(count):
        lo, hi = int(d["trace_off"][t]), int(d["trace_off"][t + 1])
        lm = int(d["trace_prof"][t])
        u[lo:hi] = oracle.predict(f[lo:hi], d["regressors"][lm])
        k[lo:hi], D[lo:hi] = oracle.key(u[lo:hi], f[lo:hi], d["profiles"][lm], r_us=d["arrival_us"][lo:hi])
    oracle.simulate(d["arrival_us"], d["true_len"], u, k, D, d["trace_off"], d["profiles"], d["trace_prof"])
    return count, time.time() - t0


def oracle_traces_timing(per_trace: int, single: int = 512, per_proc: int = 128):
    """The oracle on config-3 traces (SURVEY §8(d) Oracle (i) and (ii)): one
    thread on `single` traces, and one process per host core on `per_proc`
    traces each (disjoint trace ids); traces/s = traces / the slowest process's
    oracle seconds."""
    n1, s1 = _oracle_traces_worker((0, single, per_trace))
    procs = min(os.cpu_count() or 1, 128)  # one per host core (capped)
    # one plain subprocess per core (no multiprocessing pool: a worker that
    # fails to start must not hang the bench), each killed after 180 s
    code = ("import sys, json; sys.path.insert(0, {root!r}); import bench; "
            "print(json.dumps(bench._oracle_traces_worker(({first}, {count}, {per}))))")
    ps = [subprocess.Popen([sys.executable, "-c", code.format(root=ROOT, first=single + i * per_proc, count=per_proc,
                                                              per=per_trace)],
                           stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True) for i in range(procs)]
    res = []
    t_end = time.time() + 180
    for p in ps:
        try:
            out, _ = p.communicate(timeout=max(1.0, t_end - time.time()))
            res.append(tuple(json.loads(out.strip().splitlines()[-1])))
        except Exception:
            p.kill()
    if not res:
        raise RuntimeError("no oracle worker finished")
    tot = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return {"single_thread": {"value": round(n1 / s1, 2), "unit": "traces/s", "cores": 1, "kind": "oracle",
                              "sample": f"{single} config-3 traces x {per_trace} requests (score+key+replay)",
                              "seconds": round(s1, 3)},
            "per_core": {"value": round(tot / wall, 2), "unit": "traces/s", "cores": len(res), "kind": "oracle",
                         "host_cores": os.cpu_count(),
                         "sample": f"{len(res)} processes x {per_proc} disjoint config-3 traces x {per_trace} requests",
                         "seconds": round(wall, 3)}}


def oracle_requests_timing(d2, n_sample: int, reps: int = 1):
    """The oracle (single thread, as it stands) on a bounded sample of config 2:
    the first n_sample requests as one queue, `reps` passes (about 10-15 s)."""
    import oracle
    t0 = time.time()
    lex = oracle.Lexicon(d2["lexicon"])
    m = min(n_sample, len(d2["offsets"]) - 1)
    off = d2["offsets"][: m + 1]
    data = d2["data"][: int(off[-1])]
    t1 = time.time()
    for _ in range(reps):
        f = oracle.rule_gen(lex, data, off)
        u = oracle.predict(f, d2["regressor"])
        k, D = oracle.key(u, f, d2["profile"])
        oracle.schedule(k, u, np.asarray([0, m], np.uint32), d2["profile"])
    t2 = time.time()
    return {"value": round(m * reps / (t2 - t1) / 1e6, 5), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"config 2 queue of {m} requests (score+key+schedule) x {reps} passes, single thread",
            "seconds": round(t2 - t1, 3), "lexicon_load_s": round(t1 - t0, 4)}


# ------------------------------------------------------------------ reference arm (oracle)
def reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    import oracle
    from rtgen import configs
    m = 1 << 17
    d2 = configs.config2(n=m, gid0=0)
    lex = oracle.Lexicon(d2["lexicon"])
    seg = np.asarray([0, m], np.uint32)

    def step():
        f = oracle.rule_gen(lex, d2["data"], d2["offsets"])
        u = oracle.predict(f, d2["regressor"])
        k, D = oracle.key(u, f, d2["profile"])
        oracle.schedule(k, u, seg, d2["profile"])

    for _ in range(args.warmup):
        step()
    t0 = time.time()
    for _ in range(args.steps):
        step()
    dt = time.time() - t0
    value = m * args.steps / dt / 1e6
    sample = f"config 2 prefix queue of {m} requests per step (score+key+schedule), single thread"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8+f32", "data": "synthetic",
        "config": {"workload": "config2: one 2^20-request queue per GPU (DialoGPT profile, all r=0), "
                               "score+key+schedule", "requests_per_gpu": 1 << 20, "parallelism": "replicas1",
                   "sample": f"each step: the first {m} requests of the queue (oracle, one host thread)"},
        "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    args = parse()
    if args.impl == "reference":  # rank 0 alone (under torchrun the other ranks exit 0 without work)
        reference(args)
        return
    if args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.dry_run:
        dry_run(args)
    else:
        native(args)


if __name__ == "__main__":
    main()
