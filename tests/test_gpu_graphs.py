"""The captured-graph replay of small count calls (rs_pairwise_cardinality with
a host read-back): the graph is keyed on the batches' device arrays, the
scratch layout and the sizes, and replays with each call's own pair indices.
Repeated calls of one shape with different pairs, different ops, batches
freed and rebuilt at the same shape, and in-place run_optimize must all give
the oracle's counts."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu
OPS = ("and", "or", "andnot", "xor")


@pytest.fixture(scope="module")
def rb():
    import paper_1709_07821_b200 as p
    return p


def same_shape_images(seed, n=6, keys=8):
    """n bitmaps with the same container count (so calls on any pair share a
    graph key) but different contents and container types."""
    rng = np.random.default_rng(seed)
    imgs = []
    for i in range(n):
        vals = []
        for k in range(keys):
            kind = (i + k) % 3
            base = k << 16
            if kind == 0:    # array
                vals.append(base + rng.choice(65536, 300 + 40 * i, replace=False))
            elif kind == 1:  # bitset
                vals.append(base + rng.choice(65536, 6000 + 100 * i, replace=False))
            else:            # runs
                s = int(rng.integers(0, 60000))
                vals.append(base + np.arange(s, s + 2000 + 10 * i))
        img = orc.from_values(np.concatenate(vals).astype(np.uint64))
        imgs.append(orc.run_optimize(img)[0] if i % 2 else img)
    return imgs


def test_repeated_shape_different_pairs(rb):
    imgs = same_shape_images(1)
    B = rb.BitmapBatch.from_wire(imgs)
    pairs = [(i, j) for i in range(len(imgs)) for j in range(len(imgs))]
    for rep in range(2):
        for op in OPS:
            for i, j in pairs:
                got = B.pairwise_cardinality(op, B, [i], [j]).tolist()
                assert got == [orc.op_cardinality(op, imgs[i], imgs[j])], (rep, op, i, j)


def test_multi_pair_calls_replay(rb):
    imgs = same_shape_images(2)
    B = rb.BitmapBatch.from_wire(imgs)
    rng = np.random.default_rng(3)
    for _ in range(8):
        ia = rng.integers(0, len(imgs), 5).tolist()
        ib = rng.integers(0, len(imgs), 5).tolist()
        for op in OPS:
            want = [orc.op_cardinality(op, imgs[a], imgs[b]) for a, b in zip(ia, ib)]
            assert B.pairwise_cardinality(op, B, ia, ib).tolist() == want


def test_rebuilt_batches_and_in_place_changes(rb):
    for seed in (4, 5, 6):
        imgs = same_shape_images(seed)
        B = rb.BitmapBatch.from_wire(imgs)
        for _ in range(4):
            assert B.pairwise_cardinality("and", B, [0], [1]).tolist() == [orc.op_cardinality("and", imgs[0], imgs[1])]
        del B  # the next batch may reuse the same device blocks
    a = rb.RoaringBitmap.from_values(np.arange(0, 200000, 3, dtype=np.uint64))
    b = rb.RoaringBitmap.from_values(np.arange(0, 200000, 2, dtype=np.uint64))
    for _ in range(4):
        assert a.op_cardinality("and", b) == len(set(range(0, 200000, 3)) & set(range(0, 200000, 2)))
    a.run_optimize()
    b.run_optimize()
    for _ in range(4):
        assert a.op_cardinality("xor", b) == orc.op_cardinality("xor", a.serialize(), b.serialize())
