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


# ------------------------------------------------------- key-range sharding
# A single bitmap pair, a wide union or the all-pairs counts have too few
# independent pairs to spread, but the 2^16 chunk keys are independent
# (SURVEY 8(e)): each rank restricts its (replicated) inputs to a contiguous
# key range, computes there, and the results concatenate in key order
# (materialized results) or add up (counts: one all_reduce).

KEYS = 1 << 16


def balanced_key_ranges(hist, world: int) -> list[tuple[int, int]]:
    """Contiguous key ranges covering [0, 65536), one per rank, with about
    equal container counts (hist: containers per key)."""
    h = np.asarray(hist, dtype=np.float64)
    cum = np.concatenate([[0.0], np.cumsum(h)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")) if total else r * KEYS // world)
        cuts[-1] = min(max(cuts[-1], cuts[-2]), KEYS)
    cuts.append(KEYS)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def restrict_wire(img: bytes, lo: int, hi: int) -> bytes:
    """Host form of rs_batch_key_range on one wire image (serde.py:3-10)."""
    import struct
    (count,) = struct.unpack_from("<I", img, 4)
    desc, pays, off = [], [], 8 + 8 * count
    for k in range(count):
        key, tag, _pad, card = struct.unpack_from("<HBBI", img, 8 + 8 * k)
        size = 2 * card if tag == 1 else 8192 if tag == 2 else 2 + 4 * struct.unpack_from("<H", img, off)[0]
        if lo <= key < hi:
            desc.append(img[8 + 8 * k:16 + 8 * k])
            pays.append(img[off:off + size])
        off += size
    return b"ROAR" + struct.pack("<I", len(desc)) + b"".join(desc) + b"".join(pays)


def merge_key_ranges(parts) -> bytes:
    """Concatenate wire images whose key ranges are disjoint and ascending."""
    import struct
    desc, pays, n = [], [], 0
    for img in parts:
        (count,) = struct.unpack_from("<I", img, 4)
        n += count
        desc.append(img[8:8 + 8 * count])
        pays.append(img[8 + 8 * count:])
    return b"ROAR" + struct.pack("<I", n) + b"".join(desc) + b"".join(pays)


def _world(group):
    import torch.distributed as dist
    if not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _gather_images(img: bytes, group=None) -> list[bytes]:
    import torch.distributed as dist
    rank, world = _world(group)
    if world == 1:
        return [img]
    out = [None] * world
    dist.all_gather_object(out, img, group=group)
    return out


def _sum_counts(x: np.ndarray, group=None) -> np.ndarray:
    import torch
    import torch.distributed as dist
    rank, world = _world(group)
    if world == 1:
        return x
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64))
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()


def my_key_range(batch, group=None) -> tuple[int, int]:
    rank, world = _world(group)
    return balanced_key_ranges(batch.key_histogram(), world)[rank]


def sharded_union_many(batch, group=None) -> bytes:
    """RoaringBitmap.union_many over every bitmap of a replicated batch,
    key-range sharded; returns the union's wire image on every rank."""
    lo, hi = my_key_range(batch, group)
    local = batch.key_range(lo, hi).union_many().to_wire_list()[0]
    return merge_key_ranges(_gather_images(local, group))


def sharded_pair_op(op: str, A, B, ia: int = 0, ib: int = 0, group=None) -> bytes:
    """One bitmap pair's materialized op, key-range sharded (wire image)."""
    lo, hi = balanced_key_ranges(A.key_histogram() + B.key_histogram(), _world(group)[1])[_world(group)[0]]
    local = A.key_range(lo, hi).pairwise(op, B.key_range(lo, hi), [ia], [ib]).to_wire_list()[0]
    return merge_key_ranges(_gather_images(local, group))


def sharded_pair_count(op: str, A, B, ia: int = 0, ib: int = 0, group=None) -> int:
    """One pair's op_cardinality, key-range sharded (one all_reduce)."""
    lo, hi = balanced_key_ranges(A.key_histogram() + B.key_histogram(), _world(group)[1])[_world(group)[0]]
    c = A.key_range(lo, hi).pairwise_cardinality(op, B.key_range(lo, hi), [ia], [ib])
    return int(_sum_counts(np.asarray(c, dtype=np.int64), group)[0])


def sharded_all_pairs_cardinality(batch, group=None):
    """All-pairs |B_i and B_j|, |B_i or B_j| (config 5), key-range sharded: each
    rank's Gram tiles cover its keys; the intersection counts add up over
    ranks (one all_reduce), the unions follow from the cardinalities."""
    lo, hi = my_key_range(batch, group)
    inter, _ = batch.key_range(lo, hi).all_pairs_cardinality()
    inter = _sum_counts(np.asarray(inter, dtype=np.int64), group)
    n = len(batch)
    pi, pj = np.triu_indices(n, 1)
    card = np.asarray(batch.cardinalities(), dtype=np.int64)
    return inter, card[pi] + card[pj] - inter
