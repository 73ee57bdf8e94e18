"""N>1 host path on CPU: two gloo ranks shard bitmap pairs, gather counts, and
take the max over ranks (the GPU callback is replaced by the oracle here)."""
import os
import socket

import numpy as np
import pytest

from paper_1709_07821_b200.dist import shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 199, 1024):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from oracle import oracle as orc
    import workloads as synth
    from paper_1709_07821_b200.dist import max_over_ranks, sharded_counts
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        buf, offs = synth.config4(seed=21, nbitmaps=9, nkeys=40)
        S = orc.Session(buf, offs, 1)
        ia, ib = np.arange(8), np.arange(1, 9)
        got = sharded_counts(ia, ib, lambda a, b: S.run("or", "op_cardinality", S, a, b, 1))
        t = max_over_ranks(float(rank + 1))
        q.put((rank, got.tolist(), t))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharded_counts():
    import torch.multiprocessing as mp
    from oracle import oracle as orc
    import workloads as synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    buf, offs = synth.config4(seed=21, nbitmaps=9, nkeys=40)
    S = orc.Session(buf, offs, 1)
    want = S.run("or", "op_cardinality", S, np.arange(8), np.arange(1, 9), 1).tolist()
    for rank, got, t in res:
        assert got == want
        assert t == 2.0


# --------------------------------------------------- key-range sharding (gloo)

class OracleBatch:
    """Host stand-in for BitmapBatch in the gloo tests: the same methods the
    key-range sharding drivers call, computed by the oracle on wire images."""

    def __init__(self, images):
        self.images = list(images)

    def __len__(self):
        return len(self.images)

    def key_histogram(self):
        import struct
        h = np.zeros(1 << 16, dtype=np.uint64)
        for img in self.images:
            (n,) = struct.unpack_from("<I", img, 4)
            for k in range(n):
                h[struct.unpack_from("<H", img, 8 + 8 * k)[0]] += 1
        return h

    def key_range(self, lo, hi):
        from paper_1709_07821_b200.dist import restrict_wire
        return OracleBatch([restrict_wire(w, lo, hi) for w in self.images])

    def union_many(self):
        from oracle import oracle as orc
        return OracleBatch([orc.union_many(self.images)])

    def pairwise(self, op, other, ia, ib):
        from oracle import oracle as orc
        return OracleBatch([orc.op(op, self.images[a], other.images[b]) for a, b in zip(ia, ib)])

    def pairwise_cardinality(self, op, other, ia, ib):
        from oracle import oracle as orc
        return np.array([orc.op_cardinality(op, self.images[a], other.images[b]) for a, b in zip(ia, ib)])

    def all_pairs_cardinality(self):
        from oracle import oracle as orc
        buf = np.frombuffer(b"".join(self.images), np.uint8)
        offs = np.concatenate([[0], np.cumsum([len(w) for w in self.images])]).astype(np.uint64)
        pi, pj = np.triu_indices(len(self.images), 1)
        return orc.all_pairs_and(buf, offs, pi, pj), None

    def cardinalities(self):
        from oracle import oracle as orc
        return np.array([orc.cardinality(w) for w in self.images])

    def to_wire_list(self):
        return list(self.images)


def _images(nb=7):
    import workloads as synth
    buf, offs = synth.config4(seed=33, nbitmaps=nb, nkeys=60)
    return [buf[int(offs[i]):int(offs[i + 1])].tobytes() for i in range(nb)]


def _key_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_1709_07821_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B = OracleBatch(_images())
        out = {"union": D.sharded_union_many(B),
               "op": D.sharded_pair_op("xor", B, B, 1, 2),
               "count": D.sharded_pair_count("or", B, B, 3, 4),
               "allpairs": [x.tolist() for x in D.sharded_all_pairs_cardinality(B)],
               "range": D.my_key_range(B)}
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_key_range_sharding():
    """Key-range sharding over two gloo ranks: union_many, a
    single pair's op and count, and the all-pairs counts equal the unsharded
    results; the ranks' key ranges tile [0, 65536)."""
    import torch.multiprocessing as mp
    from oracle import oracle as orc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_key_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ws = _images()
    B = OracleBatch(ws)
    inter, _ = B.all_pairs_cardinality()
    card = B.cardinalities()
    pi, pj = np.triu_indices(len(ws), 1)
    ranges = sorted(res[r]["range"] for r in (0, 1))
    assert ranges[0][0] == 0 and ranges[0][1] == ranges[1][0] and ranges[1][1] == 1 << 16
    assert 0 < ranges[0][1] < 1 << 16  # both ranks got keys
    for r in (0, 1):
        out = res[r]
        assert out["union"] == orc.union_many(ws)
        assert out["op"] == orc.op("xor", ws[1], ws[2])
        assert out["count"] == orc.op_cardinality("or", ws[3], ws[4])
        assert out["allpairs"][0] == inter.tolist()
        assert out["allpairs"][1] == (card[pi] + card[pj] - inter).tolist()


def test_restrict_and_merge_key_ranges_roundtrip():
    from paper_1709_07821_b200.dist import balanced_key_ranges, merge_key_ranges, restrict_wire
    ws = _images(3)
    h = OracleBatch(ws).key_histogram()
    for world in (1, 2, 3, 5):
        rs = balanced_key_ranges(h, world)
        assert rs[0][0] == 0 and rs[-1][1] == 1 << 16
        for w in ws:
            assert merge_key_ranges([restrict_wire(w, lo, hi) for lo, hi in rs]) == w
