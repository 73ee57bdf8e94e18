"""Multi-GPU plumbing for the batched set operations.

The path shards with no data-path collective: bitmap pairs are independent,
so each rank (one process per GPU, torch.distributed over NCCL on GPUs, gloo
in the CPU tests) takes a contiguous range of the pair list.  Per-pair counts
are gathered to every rank with one all_gather; timing uses the max over
ranks.  Nothing here touches the GPU itself -- the per-shard work is a
callback (BitmapBatch.pairwise_cardinality on a GPU rank).
"""

from __future__ import annotations

from typing import Callable

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of n items for `rank` (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def sharded_counts(ia, ib, count_fn: Callable[[np.ndarray, np.ndarray], np.ndarray], group=None) -> np.ndarray:
    """Counts for all pairs: each rank computes its shard with count_fn, then
    one all_gather assembles the full vector on every rank."""
    import torch
    import torch.distributed as dist
    ia = np.asarray(ia, dtype=np.int64)
    ib = np.asarray(ib, dtype=np.int64)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(len(ia), rank, world)
    mine = np.asarray(count_fn(ia[lo:hi], ib[lo:hi]), dtype=np.int64)
    if world == 1:
        return mine
    sizes = [shard_range(len(ia), r, world) for r in range(world)]
    width = max(h - l for l, h in sizes)
    buf = torch.zeros(width, dtype=torch.int64)
    buf[:len(mine)] = torch.from_numpy(mine)
    if dist.get_backend(group) == "nccl":
        buf = buf.cuda()
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return np.concatenate([parts[r].cpu().numpy()[:h - l] for r, (l, h) in enumerate(sizes)])


def max_over_ranks(x: float, group=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
