"""World-size-2 gloo tests of the multi-GPU host logic: trace
sharding covers every trace exactly once, and the int64 SUM all-reduce of
per-rank statistics equals the single-process statistics exactly (the oracle
replays each rank's shard -- CPU only)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2309_06619_b200 import dist as rdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_sums(trace_ids):
    import oracle
    from rtgen import configs
    d = configs.traces(3, trace_ids, 200, lambda t: t % 4)
    lex = oracle.Lexicon(d["lexicon"])
    f = oracle.rule_gen(lex, d["data"], d["offsets"])
    n = len(d["arrival_us"])
    u = np.zeros(n, np.float32)
    k = np.zeros(n, np.uint64)
    D = np.zeros(n, np.uint32)
    for t in range(len(d["trace_off"]) - 1):
        lo, hi = d["trace_off"][t], d["trace_off"][t + 1]
        lm = int(d["trace_prof"][t])
        u[lo:hi] = oracle.predict(f[lo:hi], d["regressors"][lm])
        k[lo:hi], D[lo:hi] = oracle.key(u[lo:hi], f[lo:hi], d["profiles"][lm], r_us=d["arrival_us"][lo:hi])
    st, _ = oracle.simulate(d["arrival_us"], d["true_len"], u, k, D, d["trace_off"], d["profiles"], d["trace_prof"])
    sums = np.zeros((4, 3), np.int64)
    for t, lm in enumerate(d["trace_prof"]):
        sums[lm] += [st["sum_resp_us"][t], st["n"][t], st["misses"][t]]
    return sums


def _worker(rank, world, port, ntr, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = rdist.shard(rank, world, ntr)
        sums = torch.from_numpy(_oracle_sums(list(mine)))
        rdist.allreduce_sums(sums)
        t = rdist.max_over_ranks(float(rank + 1))
        q.put((rank, list(mine), sums.numpy(), t))
    finally:
        dist.destroy_process_group()


def test_shard_cover():
    for world in (1, 2, 3, 8):
        for n in (0, 1, 7, 4096, 65536):
            got = [i for r in range(world) for i in rdist.shard(r, world, n)]
            assert got == list(range(n))


@pytest.mark.slow
def test_allreduce_equals_single_process():
    ntr, world = 12, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, ntr, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _oracle_sums(list(range(ntr)))
    covered = sorted(i for _, mine, _, _ in res for i in mine)
    assert covered == list(range(ntr))
    for _, _, sums, t in res:
        assert (sums == want).all()      # exact integer sums, order independent
        assert t == float(world)         # MAX over ranks
    means = rdist.means_from_sums(torch.from_numpy(want))
    assert all(m > 0 for m, _ in means)


def test_bench_self_spawns_ranks_world2():
    """`python bench.py --gpus 2` without torchrun: the bench
    starts its own two ranks, which run the same process-group set-up, config-4
    block sharding, int64 SUM all-reduce and MAX-over-ranks timing as the GPU
    arm (here on gloo, --dry-run: no kernels), and rank 0 prints the line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=root, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["dry_run"] is True and line["n_gpus"] == 2 and line["backend"] == "gloo"
    assert line["config4_blocks_covered"] == [1] * 8  # every block on exactly one rank
    want = [[sum(1000 * (b + 1) + f for b in range(8)), 8 * 8192 * 1024 // 4, sum(range(8))] for f in range(4)]
    assert line["sums"] == want  # exact int64 SUM over the ranks
    assert line["ms_per_step"] >= 1.0  # the MAX over ranks saw rank 1's (+1 ms) time


def test_bench_config4_block_shards():
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for world in (1, 2, 4, 8):
        got = [b for r in range(world) for b in bench.config4_blocks(r, world)]
        assert got == list(range(8))
        assert all(len(bench.config4_blocks(r, world)) == 8 // world for r in range(world))
    with pytest.raises(ValueError):
        bench.config4_blocks(0, 3)
