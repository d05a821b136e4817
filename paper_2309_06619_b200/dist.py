"""Multi-GPU plumbing: one process per GPU, contiguous shards of
independent traces / queues, and the single collective of the path -- an int64
SUM all-reduce of the per-group statistics (row a8).  Timing is reduced with MAX
over ranks.  Works with NCCL (GPU tensors) and gloo (CPU tensors, tests)."""
from __future__ import annotations

import os


def env():
    """(rank, world_size, local_rank) from the torchrun environment."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def shard(rank: int, world: int, n: int) -> range:
    """Contiguous, balanced shard of n independent units (traces / queues)."""
    return range(rank * n // world, (rank + 1) * n // world)


def allreduce_sums(sums, group=None):
    """In-place int64 SUM of the statistics tensor (exact, order-independent)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    return sums


def max_over_ranks(x: float, device=None, group=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def means_from_sums(sums):
    """sums[g] = (sum_resp_us, n, misses) -> (mean response s, miss ratio) per group."""
    out = []
    for row in sums.tolist():
        s, n, m = row
        out.append((s / n / 1e6 if n else 0.0, m / n if n else 0.0))
    return out
