"""The one-launch single-pair path (csrc/rs_single.cu): rs_pairwise and
rs_pairwise_cardinality with one pair of bitmaps of up to 4096 result slots
run as ONE kernel (join by CTA-wide key rank, container_pairwise through the
shared bitsets, copies of unmatched keys, last-CTA compaction).  Every result
is compared byte for byte with the oracle's wire image (bitmap.py:169-241),
across container-type mixes, key overlaps (none, partial, identical), empty
sides, the largest key, the slot limit and the batched path just past it."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu
OPS = ("and", "or", "andnot", "xor")


@pytest.fixture(scope="module")
def rb():
    import paper_1709_07821_b200 as p
    return p


def bitmap(rng, keys, kinds=(0, 1, 2), optimize=False):
    """Values over the given chunk keys: per key an array, a bitset or runs."""
    vals = [np.zeros(0, dtype=np.uint64)]
    for k in keys:
        base = int(k) << 16
        kind = kinds[int(rng.integers(0, len(kinds)))]
        if kind == 0:
            v = rng.choice(65536, int(rng.integers(1, 4097)), replace=False)
        elif kind == 1:
            v = rng.choice(65536, int(rng.integers(4097, 40000)), replace=False)
        else:
            s = int(rng.integers(0, 60000))
            v = np.arange(s, s + int(rng.integers(1, 5000)))
            v = v[v < 65536]
        vals.append(base + v.astype(np.uint64))
    img = orc.from_values(np.concatenate(vals))
    return orc.run_optimize(img)[0] if optimize else img


def check_pair(rb, wa, wb, tag=""):
    B = rb.BitmapBatch.from_wire([wa, wb])
    for op in OPS:
        R = B.pairwise(op, B, [0], [1])
        assert R.to_wire_list()[0] == orc.op(op, wa, wb), (tag, op)
        assert B.pairwise_cardinality(op, B, [0], [1]).tolist() == [orc.op_cardinality(op, wa, wb)], (tag, op)
        # the result as an operand of the next call (device-only metadata)
        R2 = R.pairwise(op, B, [0], [1])
        assert R2.to_wire_list()[0] == orc.op(op, orc.op(op, wa, wb), wb), (tag, op, "chained")


@pytest.mark.parametrize("seed", range(6))
def test_random_overlaps_and_types(rb, seed):
    rng = np.random.default_rng(100 + seed)
    universe = 400
    ka = np.sort(rng.choice(universe, int(rng.integers(1, 60)), replace=False))
    kb = np.sort(rng.choice(universe, int(rng.integers(1, 60)), replace=False))
    wa = bitmap(rng, ka, optimize=seed % 2 == 0)
    wb = bitmap(rng, kb, optimize=seed % 3 == 0)
    check_pair(rb, wa, wb, seed)


def test_identical_disjoint_and_empty(rb):
    rng = np.random.default_rng(7)
    keys = np.arange(0, 40, 3)
    wa = bitmap(rng, keys)
    wb = bitmap(rng, keys)                     # same keys, other contents
    wc = bitmap(rng, keys + 1)                 # disjoint keys
    empty = orc.from_values(np.zeros(0, dtype=np.uint64))
    check_pair(rb, wa, wb, "same keys")
    check_pair(rb, wa, wa, "identical")
    check_pair(rb, wa, wc, "disjoint")
    check_pair(rb, wc, wa, "disjoint, b first")
    check_pair(rb, wa, empty, "b empty")
    check_pair(rb, empty, wa, "a empty")
    check_pair(rb, empty, empty, "both empty")


def test_largest_key_and_single_values(rb):
    top = np.array([0xFFFFFFFF, 0xFFFF0000, 0xFFFEFFFF, 0], dtype=np.uint64)
    wa = orc.from_values(top)
    wb = orc.from_values(top[:2])
    check_pair(rb, wa, wb, "top keys")
    check_pair(rb, wb, wa, "top keys, swapped")


def test_slot_limit_and_batched_fallback(rb):
    """2048 + 2048 keys (4096 slots for or / xor: the one-launch path) and
    2049 + 2048 (4097: the batched pipeline) give the oracle's results."""
    rng = np.random.default_rng(11)
    for na in (2048, 2049):
        ka = np.sort(rng.choice(8192, na, replace=False))
        kb = np.sort(rng.choice(8192, 2048, replace=False))
        wa = bitmap(rng, ka, kinds=(0, 2))
        wb = bitmap(rng, kb, kinds=(0, 2))
        B = rb.BitmapBatch.from_wire([wa, wb])
        for op in OPS:
            assert B.pairwise(op, B, [0], [1]).to_wire_list()[0] == orc.op(op, wa, wb), (na, op)
            assert B.pairwise_cardinality(op, B, [0], [1]).tolist() == [orc.op_cardinality(op, wa, wb)], (na, op)


def test_device_count_and_repeated_calls(rb):
    """Counts into device memory, and many back-to-back calls (the rotating
    completion tickets reset themselves)."""
    import torch
    rng = np.random.default_rng(12)
    wa = bitmap(rng, np.arange(0, 64))
    wb = bitmap(rng, np.arange(32, 96))
    B = rb.BitmapBatch.from_wire([wa, wb])
    dev = torch.zeros(4, dtype=torch.int64, device="cuda")
    for k, op in enumerate(OPS):
        B.pairwise_cardinality_device(op, B, dev.data_ptr() + 8 * k, 1, [0], [1])
    torch.cuda.synchronize()
    assert dev.cpu().tolist() == [orc.op_cardinality(op, wa, wb) for op in OPS]
    want = {op: orc.op(op, wa, wb) for op in OPS}
    results = [(op, B.pairwise(op, B, [0], [1])) for _ in range(150) for op in OPS]
    for op, R in results[::37]:
        assert R.to_wire_list()[0] == want[op]
    for _ in range(300):
        assert B.pairwise_cardinality("xor", B, [1], [0]).tolist() == [orc.op_cardinality("xor", wb, wa)]


def test_bitmap_class_uses_it(rb):
    rng = np.random.default_rng(13)
    va = rng.choice(1 << 22, 100_000, replace=False).astype(np.uint64)
    vb = rng.choice(1 << 22, 100_000, replace=False).astype(np.uint64)
    a, b = rb.RoaringBitmap.from_values(va), rb.RoaringBitmap.from_values(vb)
    sa, sb = set(va.tolist()), set(vb.tolist())
    assert (a & b).to_array().tolist() == sorted(sa & sb)
    assert (a | b).to_array().tolist() == sorted(sa | sb)
    assert (a - b).to_array().tolist() == sorted(sa - sb)
    assert (a ^ b).to_array().tolist() == sorted(sa ^ sb)
    assert a.op_cardinality("xor", b) == len(sa ^ sb)


def test_a_indexed_join_batches(rb):
    """AND / ANDNOT over a few pairs of many-key bitmaps take the A-indexed
    join (rs_pairwise.cu k_join_a: entries at A's container positions, no
    merged-position scans): every result against the oracle, with empty
    bitmaps, identical and disjoint pairs, and a bitmap past the shared-memory
    key limit of the per-pair join."""
    rng = np.random.default_rng(21)
    imgs = [bitmap(rng, np.sort(rng.choice(6000, k, replace=False))) for k in (700, 900, 1200, 2600)]
    imgs.append(bitmap(rng, np.arange(3000, 3700)))
    imgs.append(orc.from_values(np.zeros(0, dtype=np.uint64)))
    B = rb.BitmapBatch.from_wire(imgs)
    n = len(imgs)
    ia = [0, 1, 2, 3, 4, 5, 0, 3, 5, 2]
    ib = [1, 2, 3, 0, 0, 1, 0, 4, 5, 5]
    for op in ("and", "andnot"):
        R = B.pairwise(op, B, ia, ib)
        got = R.to_wire_list()
        for k, (a, b) in enumerate(zip(ia, ib)):
            assert got[k] == orc.op(op, imgs[a], imgs[b]), (op, a, b)
        assert R.pairwise_cardinality("or", R, list(range(len(ia))), list(range(len(ia)))).tolist() == \
            [orc.cardinality(orc.op(op, imgs[a], imgs[b])) for a, b in zip(ia, ib)]
    assert n == 6


@pytest.mark.parametrize("seed", range(3))
def test_random_batches_every_join(rb, seed):
    """Random batches whose shapes select every join: one pair (one-launch
    path), few pairs of many keys (A-indexed join for AND / ANDNOT, the
    merged-position join for OR / XOR), many pairs of few keys (per-pair
    join); pair lists with repeats and self-pairs; results and counts against
    the oracle."""
    rng = np.random.default_rng(300 + seed)
    for nbm, kmax, npairs in ((2, 80, 1), (5, 1500, 7), (40, 40, 400)):
        imgs = []
        for _ in range(nbm):
            nk = int(rng.integers(0, kmax + 1))
            imgs.append(bitmap(rng, np.sort(rng.choice(4 * kmax + 8, nk, replace=False)),
                               optimize=bool(rng.integers(0, 2))))
        B = rb.BitmapBatch.from_wire(imgs)
        ia = rng.integers(0, nbm, npairs).tolist()
        ib = rng.integers(0, nbm, npairs).tolist()
        for op in OPS:
            got = B.pairwise(op, B, ia, ib).to_wire_list()
            cnt = B.pairwise_cardinality(op, B, ia, ib).tolist()
            for k, (a, b) in enumerate(zip(ia, ib)):
                want = orc.op(op, imgs[a], imgs[b])
                assert got[k] == want, (seed, nbm, op, a, b)
                assert cnt[k] == orc.cardinality(want), (seed, nbm, op, a, b)


def test_a_indexed_join_over_per_pair_batches():
    """Per-pair-eligible AND / ANDNOT batches take the A-indexed join once
    they hold enough A containers (RS_AJOIN_MIN_SLOTS, default 32,768; config
    2's path).  Forced here on small random batches (many pairs of few keys,
    empty bitmaps, repeats and self-pairs) with RS_AJOIN_MIN_SLOTS=1, in a
    child process (the threshold is read once): results and counts against
    the oracle."""
    import os, subprocess, sys, textwrap
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = textwrap.dedent("""
        import sys
        sys.path.insert(0, %r)
        import numpy as np
        import paper_1709_07821_b200 as rb
        from oracle import oracle as orc
        from tests.test_gpu_single import bitmap
        for seed in range(3):
            rng = np.random.default_rng(700 + seed)
            for nbm, kmax, npairs in ((40, 40, 400), (12, 300, 90), (200, 16, 1500)):
                imgs = []
                for i in range(nbm):
                    nk = 0 if i == 3 else int(rng.integers(kmax // 2, kmax + 1))
                    imgs.append(bitmap(rng, np.sort(rng.choice(4 * kmax + 8, nk, replace=False)),
                                       optimize=bool(rng.integers(0, 2))))
                B = rb.BitmapBatch.from_wire(imgs)
                ia = rng.integers(0, nbm, npairs).tolist()
                ib = rng.integers(0, nbm, npairs).tolist()
                memo = {}
                for op in ("and", "andnot"):
                    got = B.pairwise(op, B, ia, ib).to_wire_list()
                    cnt = B.pairwise_cardinality(op, B, ia, ib).tolist()
                    for k, (a, b) in enumerate(zip(ia, ib)):
                        if (op, a, b) not in memo:
                            memo[(op, a, b)] = orc.op(op, imgs[a], imgs[b])
                        want = memo[(op, a, b)]
                        assert got[k] == want, (seed, nbm, op, a, b)
                        assert cnt[k] == orc.cardinality(want), (seed, nbm, op, a, b)
        print("ok")
    """) % root
    env = dict(os.environ, RS_AJOIN_MIN_SLOTS="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
