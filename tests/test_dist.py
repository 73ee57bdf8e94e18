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
