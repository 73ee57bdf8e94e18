"""GPU parity for the read/mutation paths next to the hot path:
membership (bitmap.py:99-104), for_each (:152-166), add/remove (:106-134),
memory accounting (:318-353), against the reference's golden vectors and the
reference tests' known answers (tests/test_bitmap.py)."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.golden_io import load

pytestmark = pytest.mark.gpu

CHUNK = 1 << 16


@pytest.fixture(scope="module")
def pkg():
    import paper_1709_07821_b200 as p
    return p


@pytest.fixture(scope="module")
def reference_bitmap(pkg):
    """test_bitmap.py:15-23: 1000 multiples of 62, three intervals in chunk 1,
    evens of chunk 2."""
    vals = list(range(0, 62 * 1000, 62))
    vals += list(range(CHUNK, CHUNK + 100))
    vals += list(range(CHUNK + 101, CHUNK + 201))
    vals += list(range(CHUNK + 300, CHUNK + 400))
    vals += list(range(2 * CHUNK, 3 * CHUNK, 2))
    return pkg.RoaringBitmap.from_values(vals)


def test_golden_membership_batched(pkg):
    g = load()
    bms = [g.wire(b) for b in g["mem_bm"]]
    B = pkg.BitmapBatch.from_wire(bms)
    qs = [np.frombuffer(g.wire(q), dtype="<u4") for q in g["mem_q"]]
    want = np.concatenate([np.frombuffer(g.wire(h), dtype=np.uint8).astype(bool) for h in g["mem_hit"]])
    idx = np.concatenate([np.full(len(q), i, dtype=np.uint32) for i, q in enumerate(qs)])
    got = B.contains(np.concatenate(qs), idx)
    assert np.array_equal(got, want)
    for i, (w, q) in enumerate(zip(bms, qs)):  # the one-bitmap API agrees
        rb = pkg.RoaringBitmap.deserialize(w)
        assert np.array_equal(rb.contains_many(q), want[idx == i])


def test_golden_add_remove_sequences(pkg):
    g = load()
    m = g["mut"]
    for start, ops, changed, imgs in zip(g["mut_start"], m["ops"], m["changed"], m["img"]):
        rb = pkg.RoaringBitmap.deserialize(g.wire(start))
        for (kind, v), ch, img in zip(ops, changed, imgs):
            got = rb.add(v) if kind == "add" else rb.remove(v)
            assert int(got) == ch, (kind, v)
            assert rb.serialize() == g.wire(img), (kind, v)


def test_membership_random_vs_oracle(pkg):
    rng = np.random.default_rng(99)
    wires = []
    for t in range(12):
        vals = np.unique(rng.integers(0, 6 * CHUNK, size=int(rng.integers(0, 60000)))).astype(np.uint64)
        w = orc.from_values(vals)
        if t % 2:
            w = orc.run_optimize(w)[0]
        wires.append(w)
    B = pkg.BitmapBatch.from_wire(wires)
    q = rng.integers(0, 7 * CHUNK, size=200000).astype(np.uint32)
    bi = rng.integers(0, len(wires), size=q.size).astype(np.uint32)
    got = B.contains(q, bi)
    want = np.zeros(q.size, dtype=bool)
    for i, w in enumerate(wires):
        sel = bi == i
        want[sel] = np.isin(q[sel], orc.to_array(w))
    assert np.array_equal(got, want)


def test_reference_membership_and_for_each(pkg, reference_bitmap):
    rb = reference_bitmap
    assert 62 in rb                                   # test_bitmap.py:26-31
    assert CHUNK + 100 not in rb
    assert (2 * CHUNK) + 1 not in rb
    assert 2 * CHUNK in rb
    assert -1 not in rb and (1 << 32) not in rb
    assert rb.for_each(lambda v: True) == 1000 + 300 + 32768   # test_bitmap.py:34-38
    assert rb.for_each(lambda v: False) == 1
    assert pkg.RoaringBitmap().for_each(lambda v: True) == 0
    seen = []
    rb.for_each(lambda v: seen.append(v) or len(seen) < 5)
    assert seen == [0, 62, 124, 186, 248]


def test_add_remove_chunks(pkg):
    rb = pkg.RoaringBitmap()                          # test_bitmap.py:53-64
    assert rb.add(1 << 31)
    assert [k for k, _ in rb.chunks()] == [0x8000]
    c = next(c for _, c in rb.chunks())
    assert isinstance(c, pkg.ArrayContainer) and c.values.tolist() == [0]
    assert not rb.add(1 << 31)
    assert rb.remove(1 << 31)
    assert len(rb) == 0 and not list(rb.chunks())
    for v in range(4097):
        rb.add(v)
    assert isinstance(next(c for _, c in rb.chunks()), pkg.BitsetContainer)
    with pytest.raises(ValueError):
        rb.add(1 << 32)
    assert not rb.remove(1 << 32) and not rb.remove(-5)


def test_memory_accounting(pkg, reference_bitmap):
    RB = pkg.RoaringBitmap
    assert RB().memory_bytes() == (16, 8)             # test_bitmap.py:171-177
    mem, ser = RB.from_values(range(2 * CHUNK, 3 * CHUNK, 2)).memory_bytes()
    assert mem == 16 + 7 + 8192
    assert RB.from_values([0]).memory_bytes() == (16 + 7 + 2, 8 + 8 + 2)
    rb = reference_bitmap.copy()
    rb.run_optimize()
    assert rb.memory_bytes()[1] == len(rb.serialize())   # test_serde.py:78
    # array 1000 values, run of 3 runs, bitset
    assert rb.memory_bytes()[0] == 16 + 3 * 7 + 2000 + 12 + 8192


def test_run_optimize_and_shrink_never_grow_memory(pkg):
    rng = np.random.default_rng(8)                    # test_bitmap.py:153-168
    rb = pkg.RoaringBitmap()
    for v in rng.integers(0, 1 << 18, size=300).tolist():
        rb.add(int(v))
    for s in range(200000, 200300):
        rb.add(s)
    before_mem, _ = rb.memory_bytes()
    before = rb.to_array()
    rb.run_optimize()
    reclaimed = rb.shrink_to_fit()
    after_mem, _ = rb.memory_bytes()
    assert reclaimed >= 0 and after_mem <= before_mem
    assert np.array_equal(rb.to_array(), before)
    rb.validate()


# ---------------------------------------- container-level element functions
# test_containers.py:55-135 known answers (container_add/remove/contains/normalize)

def _arr(pkg, vals):
    return pkg.ArrayContainer(np.array(sorted(vals), dtype=np.uint16))


def _run(pkg, ivs):
    return pkg.RunContainer(np.array(ivs, dtype=np.uint16))


def _bitset(pkg, vals):
    w = np.zeros(1024, dtype=np.uint64)
    for v in vals:
        w[v >> 6] |= np.uint64(1) << np.uint64(v & 63)
    return pkg.BitsetContainer(w, len(vals))


def test_container_add_remove_contains(pkg):
    c, changed = pkg.container_add(_arr(pkg, [1, 3, 5]), 7)
    assert changed and c.values.tolist() == [1, 3, 5, 7]
    c, changed = pkg.container_add(_arr(pkg, [1, 3, 5]), 3)
    assert not changed and c.values.tolist() == [1, 3, 5]
    full = pkg.ArrayContainer(np.arange(4096, dtype=np.uint16))
    c, changed = pkg.container_add(full, 4096)
    assert changed and isinstance(c, pkg.BitsetContainer) and len(c) == 4097
    c, changed = pkg.container_remove(_arr(pkg, [1, 3, 5]), 3)
    assert changed and c.values.tolist() == [1, 5]
    big = _bitset(pkg, range(4097))
    c, changed = pkg.container_remove(big, 17)
    assert changed and isinstance(c, pkg.ArrayContainer) and len(c) == 4096
    r, changed = pkg.container_remove(_run(pkg, [(100, 100)]), 150)
    assert changed and isinstance(r, pkg.RunContainer)
    assert r.runs.tolist() == [[100, 49], [151, 49]]
    r = _run(pkg, [(0, 99), (101, 99), (300, 99)])
    assert not pkg.container_contains(r, 100) and pkg.container_contains(r, 200)
    b = _bitset(pkg, [0] + list(range(100, 4200)))
    assert pkg.container_contains(b, 0) and not pkg.container_contains(b, 1)
    base = pkg.ArrayContainer(np.arange(4096, dtype=np.uint16))
    c, _ = pkg.container_add(base.copy(), 5000)
    assert isinstance(c, pkg.BitsetContainer)
    c, _ = pkg.container_remove(c, 5000)
    assert c == base


def test_container_normalize_rules(pkg):
    evens = _run(pkg, [(v, 0) for v in range(0, 65536, 2)])
    n = pkg.container_normalize(evens)
    assert isinstance(n, pkg.BitsetContainer) and len(n) == 32768
    one_run = _run(pkg, [(0, 999)])
    assert pkg.container_normalize(one_run) is one_run
    assert len(pkg.container_normalize(pkg.ArrayContainer())) == 0
    n = pkg.container_normalize(_run(pkg, [(0, 1), (10, 1)]))   # strict tie goes to the array
    assert isinstance(n, pkg.ArrayContainer) and n.values.tolist() == [0, 1, 10, 11]
    c = _arr(pkg, range(0, 1000))
    assert pkg.container_normalize(c) is c
    opt = pkg.container_normalize(c, consider_run=True)
    assert isinstance(opt, pkg.RunContainer) and opt.runs.tolist() == [[0, 999]]
    r = _run(pkg, [(i * 4, 1) for i in range(3000)])             # 6000 values, 3000 runs
    assert isinstance(pkg.container_normalize(r), pkg.BitsetContainer)
    r = _run(pkg, [(i * 32, 20) for i in range(2000)])           # 42000 values, 2000 runs
    assert pkg.container_normalize(r) is r
