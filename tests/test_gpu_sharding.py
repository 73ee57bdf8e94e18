"""Multi-GPU building blocks on one GPU: rs_batch_key_range / key_histogram
against their host definitions, and the key-range sharded drivers
(paper_1709_07821_b200/dist.py) at world size 1 against the unsharded ops.
(The N-rank collectives are covered with gloo on CPU: tests/test_dist.py.)"""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def test_key_range_matches_host_restriction():
    import paper_1709_07821_b200 as rb
    from paper_1709_07821_b200.dist import balanced_key_ranges, merge_key_ranges, restrict_wire
    import workloads as synth
    buf, offs = synth.config4(seed=7, nbitmaps=12, nkeys=300)
    ws = [buf[int(offs[i]):int(offs[i + 1])].tobytes() for i in range(12)]
    B = rb.BitmapBatch.from_wire(ws)
    h = B.key_histogram()
    assert int(h.sum()) == int(B.container_counts().sum())
    for lo, hi in balanced_key_ranges(h, 3) + [(0, 0), (100, 40000), (0, 65536)]:
        R = B.key_range(lo, hi)
        assert R.to_wire_list() == [restrict_wire(w, lo, hi) for w in ws], (lo, hi)
        assert np.array_equal(R.digests(), rb.BitmapBatch.from_wire([restrict_wire(w, lo, hi) for w in ws]).digests())
    parts = [B.key_range(lo, hi).to_wire_list() for lo, hi in balanced_key_ranges(h, 4)]
    assert [merge_key_ranges([p[i] for p in parts]) for i in range(12)] == ws


def test_sharded_drivers_single_rank():
    import paper_1709_07821_b200 as rb
    from paper_1709_07821_b200 import dist as D
    import workloads as synth
    buf, offs = synth.config4(seed=8, nbitmaps=10, nkeys=200)
    ws = [buf[int(offs[i]):int(offs[i + 1])].tobytes() for i in range(10)]
    B = rb.BitmapBatch.from_wire(ws)
    assert D.sharded_union_many(B) == orc.union_many(ws)
    assert D.sharded_pair_op("andnot", B, B, 2, 5) == orc.op("andnot", ws[2], ws[5])
    assert D.sharded_pair_count("xor", B, B, 2, 5) == orc.op_cardinality("xor", ws[2], ws[5])
    inter, uni = D.sharded_all_pairs_cardinality(B)
    pi, pj = np.triu_indices(10, 1)
    assert np.array_equal(inter, orc.all_pairs_and(buf, offs, pi, pj))
