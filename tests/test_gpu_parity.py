"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the C oracle, byte for byte on wire images (values + container
types) and exactly on counts."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.golden_io import load

pytestmark = pytest.mark.gpu

OPS = ("and", "or", "andnot", "xor")


@pytest.fixture(scope="module")
def pkg():
    import paper_1709_07821_b200 as p
    return p


def _wires(buf, offs):
    return [buf[int(offs[i]):int(offs[i + 1])].tobytes() for i in range(len(offs) - 1)]


# ------------------------------------------------------------ golden vectors

def test_golden_pairs_batched(pkg):
    g = load()
    A = pkg.BitmapBatch.from_wire([g.wire(a) for a in g["pair_a"]])
    B = pkg.BitmapBatch.from_wire([g.wire(b) for b in g["pair_b"]])
    for k, op in enumerate(OPS):
        got = A.pairwise(op, B).to_wire_list()
        want = [g.wire(r[k]) for r in g["pair_res"]]
        bad = [i for i, (x, y) in enumerate(zip(got, want)) if x != y]
        assert not bad, (op, bad[:5])
        cards = A.pairwise_cardinality(op, B)
        assert cards.tolist() == [int(c[k]) for c in g["pair_card"]], op


def test_golden_container_pairs(pkg):
    g = load()
    A = pkg.BitmapBatch.from_wire([g.wire(a) for a in g["cont_a"]])
    B = pkg.BitmapBatch.from_wire([g.wire(b) for b in g["cont_b"]])
    for k, op in enumerate(OPS):
        got = A.container_pairwise(op, B).to_wire_list()
        want = [g.wire(r[k]) for r in g["cont_res"]]
        bad = [(i, tuple(g["cont_tags"][i])) for i, (x, y) in enumerate(zip(got, want)) if x != y]
        assert not bad, (op, bad[:5])
        cards = A.container_pairwise_cardinality(op, B)
        assert cards.tolist() == [int(c[k]) for c in g["cont_card"]], op


def test_golden_union_many(pkg):
    g = load()
    for members, res in zip(g["um_members"], g["um_res"]):
        ws = [g.wire(m) for m in members]
        if not ws:
            assert pkg.RoaringBitmap.union_many([]) == pkg.RoaringBitmap()
            continue
        got = pkg.BitmapBatch.from_wire(ws).union_many().to_wire_list()[0]
        assert got == g.wire(res)


def test_golden_from_values_run_optimize_to_array(pkg):
    g = load()
    buf, off = g["fv_in_buf"], g["fv_in_off"]
    arrays = [np.frombuffer(buf[int(off[i]):int(off[i + 1])].tobytes(), dtype="<u8")
              for i in range(len(off) - 1)]
    B = pkg.BitmapBatch.from_values(arrays)
    assert B.to_wire_list() == [g.wire(r) for r in g["fv_res"]]
    vals = B.to_arrays()
    for v, a in zip(vals, g["fv_arr"]):
        assert v.astype("<u4").tobytes() == g.wire(a)
    changed = B.run_optimize()
    assert changed.tolist() == [bool(c) for c in g["fv_changed"]]
    assert B.to_wire_list() == [g.wire(r) for r in g["fv_opt"]]


def test_golden_decode_errors(pkg):
    g = load()
    for img, off, msg in zip(g["bad"], g["bad_off"], g["bad_msg"]):
        with pytest.raises(pkg.DecodeError) as e:
            pkg.BitmapBatch.from_wire([g.wire(img)])
        assert e.value.offset == off and str(e.value) == msg


# ------------------------------------------------ reference API known answers

def test_bitmap_api_known_answers(pkg):
    RB = pkg.RoaringBitmap
    a = RB.from_values([1, 3, 5, 7])
    b = RB.from_values([1, 2, 3, 4, 6, 7, 8, 9])
    assert [a.op_cardinality(op, b) for op in OPS] == [3, 9, 1, 6]   # test_bitmap.py:78-85
    assert a.op_cardinality("andnot", a) == 0
    a = RB.from_values([5, 70000, 200000])
    b = RB.from_values([5, 200000, 999999])
    assert (a & b).to_array().tolist() == [5, 200000]                 # test_bitmap.py:88-95
    assert (a | b).to_array().tolist() == [5, 70000, 200000, 999999]
    assert (a - b).to_array().tolist() == [70000]
    assert (a ^ b).to_array().tolist() == [70000, 999999]
    assert list(a) == [5, 70000, 200000]
    e = RB()
    assert len(e) == 0 and not e and e.to_array().size == 0
    x = RB.from_values([1, 2, 3])
    assert x.op("or", RB()) == x and len(x.op("xor", x)) == 0
    with pytest.raises(ValueError):
        x.op("nand", x)
    with pytest.raises(ValueError):
        RB.from_values([1, 1 << 32])
    before = x.copy()
    for op in OPS:
        x.op(op, a)
        x.op_cardinality(op, a)
    assert x == before                                                # inputs never mutated


def test_container_level_conversions(pkg):
    # test_containers.py:160-170: on-the-fly type conversion
    lo = pkg.BitsetContainer(np.zeros(1024, np.uint64), 0)
    lo = pkg.RoaringBitmap.from_values(range(5000))
    hi = pkg.RoaringBitmap.from_values(range(4000, 9000))
    (_, A), = list(lo.chunks())
    (_, B), = list(hi.chunks())
    inter = pkg.container_pairwise("and", A, B)
    assert isinstance(inter, pkg.ArrayContainer) and len(inter) == 1000
    union = pkg.container_pairwise("or", A, B)
    assert isinstance(union, pkg.BitsetContainer) and len(union) == 9000
    wa = pkg.ArrayContainer(np.arange(0, 8000, 2, dtype=np.uint16))
    wb = pkg.ArrayContainer(np.arange(1, 8000, 2, dtype=np.uint16))
    u = pkg.container_pairwise("or", wa, wb)
    assert isinstance(u, pkg.BitsetContainer) and len(u) == 8000
    assert pkg.container_pairwise_cardinality("xor", wa, wa) == 0


# ------------------------------------------------ synthetic configs vs oracle

def _check_pairs(pkg, wa, wb, A, B, ia, ib, ops=OPS, sample=None):
    idx = np.arange(len(ia)) if sample is None else sample
    for op in ops:
        R = A.pairwise(op, B, ia, ib)
        got = R.to_wire_list()
        for p in idx:
            assert got[p] == orc.op(op, wa[ia[p]], wb[ib[p]]), (op, int(p))
        cards = A.pairwise_cardinality(op, B, ia, ib)
        want = [orc.op_cardinality(op, wa[ia[p]], wb[ib[p]]) for p in range(len(ia))]
        assert cards.tolist() == want, op
        assert R.cardinalities().tolist() == want, op


def test_config1_full(pkg):
    import workloads as synth
    buf, offs = synth.config1()
    w = _wires(buf, offs)
    Bt = pkg.BitmapBatch.from_wire((buf, offs))
    _check_pairs(pkg, w, w, Bt, Bt, [0], [1])


def test_config2_subset(pkg):
    import workloads as synth
    buf, offs = synth.config2(npairs=24)
    w = _wires(buf, offs)
    Bt = pkg.BitmapBatch.from_wire((buf, offs))
    ia, ib = list(range(24)), list(range(24, 48))
    _check_pairs(pkg, w, w, Bt, Bt, ia, ib)


def test_config3_subset(pkg):
    import workloads as synth
    n = 30000
    buf, offs = synth.config3(npairs=n)
    A = pkg.BitmapBatch.from_wire(synth.slice_images(buf, offs, 0, n))
    B = pkg.BitmapBatch.from_wire(synth.slice_images(buf, offs, n, 2 * n))
    bA, oA = synth.slice_images(buf, offs, 0, n)
    bB, oB = synth.slice_images(buf, offs, n, 2 * n)
    idx = np.arange(n)
    for op in OPS:
        got = A.container_pairwise(op, B).to_wire_list()
        bufA, offA = orc.concat([bA[int(oA[i]):int(oA[i + 1])].tobytes() for i in range(n)])
        want = orc.op_batch(op, bufA, offA, *orc.concat([bB[int(oB[i]):int(oB[i + 1])].tobytes() for i in range(n)]),
                            idx, idx)
        bad = [i for i in range(n) if got[i] != want[i]]
        assert not bad, (op, bad[:5])
        cards = A.container_pairwise_cardinality(op, B)
        wc = orc.container_card_batch(op, bufA, offA, *orc.concat(
            [bB[int(oB[i]):int(oB[i + 1])].tobytes() for i in range(n)]), idx, idx)
        assert np.array_equal(cards.astype(np.int64), wc), op


def test_config4_subset_pairs_and_union(pkg):
    import workloads as synth
    nb = 10
    buf, offs = synth.config4(nbitmaps=nb)
    w = _wires(buf, offs)
    Bt = pkg.BitmapBatch.from_wire((buf, offs))
    ia, ib = list(range(nb - 1)), list(range(1, nb))
    _check_pairs(pkg, w, w, Bt, Bt, ia, ib)
    assert Bt.union_many().to_wire_list()[0] == orc.union_many(w)


def test_config5_subset_all_pairs(pkg):
    import workloads as synth
    nb = 20
    buf, offs = synth.config5(nbitmaps=nb)
    Bt = pkg.BitmapBatch.from_wire((buf, offs))
    inter, uni = Bt.all_pairs_cardinality()
    pi, pj = np.triu_indices(nb, 1)
    want = orc.all_pairs_and(buf, offs, pi, pj)
    assert np.array_equal(inter.astype(np.int64), want)
    cards = Bt.cardinalities().astype(np.int64)
    assert np.array_equal(uni.astype(np.int64), cards[pi] + cards[pj] - want)


def _all_pairs_check(pkg, buf, offs):
    Bt = pkg.BitmapBatch.from_wire((buf, offs))
    nb = len(offs) - 1
    inter, uni = Bt.all_pairs_cardinality()
    pi, pj = np.triu_indices(nb, 1)
    want = orc.all_pairs_and(buf, offs, pi, pj)
    assert np.array_equal(inter.astype(np.int64), want)
    cards = Bt.cardinalities().astype(np.int64)
    assert np.array_equal(uni.astype(np.int64), cards[pi] + cards[pj] - want)


def test_all_pairs_tensor_core_tiles(pkg, monkeypatch):
    """The tcgen05 Gram tiles (k_allpairs_umma) on every key, including a key
    with 300 containers (3 x 3 tile blocks, off-diagonal tiles), against the
    oracle's pairwise intersections; and the CUDA-core tiles for the same
    input."""
    import workloads as synth
    rng = np.random.default_rng(77)
    imgs = []
    for i in range(300):  # one container at key 0 per bitmap: m = 300 for that key
        kind = i % 3
        if kind == 0:
            v = rng.choice(65536, int(rng.integers(1, 4000)), replace=False)
        elif kind == 1:
            v = np.nonzero(rng.random(65536) < rng.uniform(0.1, 0.9))[0]
        else:
            s = int(rng.integers(0, 60000))
            v = np.arange(s, s + int(rng.integers(1, 5000)))
        extra = rng.choice(np.arange(1, 8), 2, replace=False) * 65536 + rng.integers(0, 65536, 2)
        w = orc.from_values(np.concatenate([v, extra]).astype(np.uint64))
        imgs.append(orc.run_optimize(w)[0] if i % 5 == 0 else w)
    offs = np.zeros(len(imgs) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(x) for x in imgs])
    buf = np.frombuffer(b"".join(imgs), dtype=np.uint8)
    monkeypatch.setenv("RS_ALLPAIRS_UMMA_MIN", "2")
    _all_pairs_check(pkg, buf, offs)
    b5, o5 = synth.config5(nbitmaps=160)
    _all_pairs_check(pkg, b5, o5)
    monkeypatch.setenv("RS_ALLPAIRS_UMMA", "0")
    _all_pairs_check(pkg, buf, offs)


def test_run_optimize_matches_oracle(pkg):
    import workloads as synth
    buf, offs = synth.config5(nbitmaps=6, seed=9)
    # strip runs first: re-build from values, then run_optimize on the GPU
    Bt = pkg.BitmapBatch.from_wire((buf, offs))
    V = pkg.BitmapBatch.from_values(Bt.to_arrays())
    ch = V.run_optimize()
    for i, w in enumerate(V.to_wire_list()):
        ref, rch = orc.run_optimize(orc.from_values(Bt.to_arrays()[i]))
        assert w == ref and ch[i] == rch


def test_edge_cases(pkg):
    RB = pkg.RoaringBitmap
    empty = RB()
    full = RB.from_values(np.arange(0, 1 << 17, dtype=np.uint32))   # two full bitset chunks
    full.run_optimize()
    one = RB.from_values([65535])
    cases = [empty, full, one, RB.from_values([0, 65535, 65536, (1 << 32) - 1])]
    ws = [c.serialize() for c in cases]
    for a, wa in zip(cases, ws):
        for b, wb in zip(cases, ws):
            for op in OPS:
                assert a.op(op, b).serialize() == orc.op(op, wa, wb), op
                assert a.op_cardinality(op, b) == orc.op_cardinality(op, wa, wb)


def test_exact_and_upper_bound_allocation_agree(pkg, monkeypatch):
    """Both result-pool sizing modes (host-synchronized exact sizes vs. the
    no-sync upper bound) produce identical bitmaps."""
    g = load()
    A = pkg.BitmapBatch.from_wire([g.wire(a) for a in g["pair_a"]])
    B = pkg.BitmapBatch.from_wire([g.wire(b) for b in g["pair_b"]])
    for op in OPS:
        monkeypatch.setenv("RS_EXACT_ALLOC", "1")
        exact = A.pairwise(op, B).to_wire_list()
        monkeypatch.setenv("RS_EXACT_ALLOC", "0")
        fast = A.pairwise(op, B).to_wire_list()
        assert exact == fast == [g.wire(r[OPS.index(op)]) for r in g["pair_res"]]


def test_harness_rows_gate_and_format(pkg):
    import io
    from paper_1709_07821_b200 import harness
    import workloads as synth
    buf, offs = synth.config4(seed=31, nbitmaps=5, nkeys=50)
    B = pkg.BitmapBatch.from_wire((buf, offs))
    S = orc.Session(buf, offs)
    ia, ib = np.arange(4), np.arange(1, 5)
    rows = harness.bench_pairwise("c4mini", B, "or", S.run("or", "op", S, ia, ib))
    rows += harness.bench_pairwise("c4mini", B, "and", S.run("and", "op_cardinality", S, ia, ib), count_only=True)
    rep = harness.BenchReport(rows)
    out = io.StringIO()
    rep.to_csv(out)
    assert out.getvalue().splitlines()[0] == ",".join(harness.CSV_COLUMNS)
    assert [r.metric for r in rows] == ["or", "and_count"] and all(r.value > 0 for r in rows)
    with pytest.raises(harness.CorrectnessError):
        harness.bench_pairwise("c4mini", B, "xor", np.zeros(4, dtype=np.int64))


# ---------------------------------------------- deferred (asynchronous) ingest

def test_deferred_ingest_golden_pairs(pkg):
    g = load()
    A = pkg.BitmapBatch.from_wire([g.wire(a) for a in g["pair_a"]], deferred=True)
    B = pkg.BitmapBatch.from_wire([g.wire(b) for b in g["pair_b"]], deferred=True)
    for k, op in enumerate(OPS):  # ops queued before the checks are read back
        got = A.pairwise(op, B).to_wire_list()
        assert got == [g.wire(r[k]) for r in g["pair_res"]], op
    A.wait()
    B.wait()


def test_deferred_ingest_decode_errors(pkg):
    """Every golden DecodeError surfaces with the reference's offset and
    message: structural ones at from_wire, payload ones at wait() or at the
    first host readback; ops queued on a failing batch stay in bounds."""
    g = load()
    good = pkg.BitmapBatch.from_wire([g.wire(g["pair_a"][0])])
    for img, off, msg in zip(g["bad"], g["bad_off"], g["bad_msg"]):
        try:
            b = pkg.BitmapBatch.from_wire([g.wire(img)], deferred=True)
        except pkg.DecodeError as e:
            assert e.offset == off and str(e) == msg
            continue
        for op in OPS:  # queued before the checks are known
            b.pairwise(op, good)
        with pytest.raises(pkg.DecodeError):  # host readback resolves the checks
            b.pairwise_cardinality("and", good)
        with pytest.raises(pkg.DecodeError) as e:
            b.wait()
        assert e.value.offset == off and str(e.value) == msg
        with pytest.raises(pkg.DecodeError):
            b.to_wire_list()
        with pytest.raises(pkg.DecodeError):
            b.wait()


def test_deferred_ingest_pipeline_matches_sync(pkg):
    """Chunked ingest on the copy stream overlapping ops on the library
    stream (the e2e pattern of bench.py) gives the synchronous results."""
    from paper_1709_07821_b200 import _lib
    import workloads as synth
    buf, offs = synth.config2(npairs=32)
    n = 32
    pin = _lib.PinnedBuffer(int(offs[-1]))
    pin.array[:] = buf[:int(offs[-1])]
    A_sync = pkg.BitmapBatch.from_wire((buf[:int(offs[n])], offs[:n + 1].copy()))
    B_sync = pkg.BitmapBatch.from_wire((buf[int(offs[n]):], offs[n:] - offs[n]))
    want = {op: A_sync.pairwise(op, B_sync).to_wire_list() for op in OPS}
    got = {op: [] for op in OPS}
    batches = []
    step = 8
    for p0 in range(0, n, step):
        def part(base, p0=p0):
            o = offs[base + p0:base + p0 + step + 1]
            return (pin.array[int(o[0]):int(o[-1])], (o - o[0]).astype(np.uint64))
        A = pkg.BitmapBatch.from_wire(part(0), deferred=True)
        B = pkg.BitmapBatch.from_wire(part(n), deferred=True)
        batches += [A, B]
        for op in OPS:
            got[op].append(A.pairwise(op, B))
    for b in batches:
        b.wait()
    for op in OPS:
        assert [w for R in got[op] for w in R.to_wire_list()] == want[op], op


def test_deferred_ingest_lifecycle(pkg):
    """Deferred batches freed before first use hand their staging slot back;
    many in flight at once; pageable input; a run container that can never be
    admissible (> 2047 runs) takes the synchronous path and raises at once."""
    g = load()
    imgs = [g.wire(a) for a in g["pair_a"]]
    want = pkg.BitmapBatch.from_wire(imgs).to_wire_list()
    for _ in range(3):  # created and dropped unused: slots must come back
        pkg.BitmapBatch.from_wire(imgs, deferred=True)
    live = [pkg.BitmapBatch.from_wire(imgs, deferred=True) for _ in range(12)]
    for b in live:
        assert b.to_wire_list() == want
        b.wait()
    # > 2047 runs in one container: structurally valid, never admissible
    runs = np.arange(0, 2 * 2100, 2, dtype=np.uint16)
    img = (b"ROAR" + (1).to_bytes(4, "little") + (0).to_bytes(2, "little") + bytes([3, 0]) +
           len(runs).to_bytes(4, "little") + len(runs).to_bytes(2, "little") +
           np.stack([runs, np.zeros_like(runs)], 1).astype("<u2").tobytes())
    with pytest.raises(pkg.DecodeError) as e:
        pkg.BitmapBatch.from_wire([img], deferred=True)
    with pytest.raises(pkg.DecodeError) as e2:
        pkg.BitmapBatch.from_wire([img])
    assert str(e.value) == str(e2.value) and e.value.offset == e2.value.offset


def test_contains_edge_cases(pkg):
    B = pkg.BitmapBatch.from_values([np.array([0, 65535, 65536, 1 << 31, 0xFFFFFFFF], dtype=np.uint64),
                                     np.array([], dtype=np.uint64)])
    q = [0, 1, 65535, 65536, 65537, 1 << 31, 0xFFFFFFFF, 0xFFFFFFFE]
    assert B.contains(q).tolist() == [True, False, True, True, False, True, True, False]
    assert B.contains(q, [1] * len(q)).tolist() == [False] * len(q)
    assert B.contains([]).size == 0
    with pytest.raises(Exception):
        B.contains([1], [2])          # bitmap index out of range
    with pytest.raises(ValueError):
        B.contains([1 << 32])


def test_random_pairs_vs_oracle(pkg):
    """test_bitmap.py::test_ops_match_oracle_random, batched: 240 seeded random
    pairs (universes from 100 values to 2^21, sizes 0..12000, a third of them
    run-optimized so runs meet arrays and bitsets) through the four ops and
    their counts, byte for byte against the oracle."""
    rng = np.random.default_rng(20261019)
    wa, wb = [], []
    for i in range(240):
        universe = int(rng.integers(100, 1 << 21))
        ws = []
        for _ in range(2):
            n = int(rng.integers(0, 12000))
            if rng.random() < 0.3:  # clustered: long runs
                start = int(rng.integers(0, universe))
                v = np.arange(start, start + n, dtype=np.uint64)
            else:
                v = np.unique(rng.integers(0, universe, size=n)).astype(np.uint64)
            w = orc.from_values(v)
            ws.append(orc.run_optimize(w)[0] if i % 3 == 0 else w)
        wa.append(ws[0])
        wb.append(ws[1])
    A = pkg.BitmapBatch.from_wire(wa)
    B = pkg.BitmapBatch.from_wire(wb)
    for op in OPS:
        got = A.pairwise(op, B).to_wire_list()
        bad = [i for i in range(len(wa)) if got[i] != orc.op(op, wa[i], wb[i])]
        assert not bad, (op, bad[:5])
        cards = A.pairwise_cardinality(op, B).tolist()
        assert cards == [orc.op_cardinality(op, x, y) for x, y in zip(wa, wb)], op


def test_maximum_key_counts(pkg):
    """Bitmaps spanning all 65,536 chunk keys (one value per chunk, or full
    chunks as single runs) against sparse ones: the key join's global-memory
    path (more than 2,048 containers per bitmap), 65,536-entry results, and
    full-chunk runs, byte for byte against the oracle."""
    rng = np.random.default_rng(65536)
    every_key = (np.arange(65536, dtype=np.uint64) << 16) + rng.integers(0, 65536, 65536).astype(np.uint64)
    w_every = orc.from_values(every_key)
    full_chunks = np.concatenate([np.arange(k << 16, (k + 1) << 16, dtype=np.uint64)
                                  for k in rng.choice(65536, 24, replace=False)])
    w_full = orc.run_optimize(orc.from_values(full_chunks))[0]
    w_sparse = orc.from_values(np.unique(rng.integers(0, 1 << 32, 5000)).astype(np.uint64))
    ws = [w_every, w_full, w_sparse]
    A = pkg.BitmapBatch.from_wire(ws)
    ia, ib = [0, 0, 1, 2, 1], [1, 2, 2, 0, 0]
    for op in OPS:
        got = A.pairwise(op, A, ia, ib).to_wire_list()
        for k, (a, b) in enumerate(zip(ia, ib)):
            assert got[k] == orc.op(op, ws[a], ws[b]), (op, a, b)
        cards = A.pairwise_cardinality(op, A, ia, ib).tolist()
        assert cards == [orc.op_cardinality(op, ws[a], ws[b]) for a, b in zip(ia, ib)], op
    assert np.array_equal(A.to_arrays()[0], np.sort(every_key).astype(np.uint32))


@pytest.mark.parametrize("npairs", [1, 4096, 4097])
def test_scan_over_pairs_fused_and_separate(pkg, npairs):
    """The per-pair join scans over pairs inside k_merge_pair / k_pair_nonempty
    (last-CTA pattern) up to 4096 pairs and with separate scan launches above:
    both sides of the boundary, byte for byte against the oracle.  Small seeded
    bitmaps (a few chunks each, some pairs with empty results so per-pair
    compaction drops entries)."""
    rng = np.random.default_rng(4097 + npairs)
    pool = []
    for _ in range(64):
        keys = rng.choice(24, size=int(rng.integers(1, 6)), replace=False)
        v = np.concatenate([(int(k) << 16) + np.unique(rng.integers(0, 1 << 16, size=int(rng.integers(1, 6000))))
                            for k in keys]).astype(np.uint64)
        pool.append(orc.from_values(np.sort(v)))
    ia = rng.integers(0, 64, size=npairs).astype(np.uint32)
    ib = rng.integers(0, 64, size=npairs).astype(np.uint32)
    P = pkg.BitmapBatch.from_wire(pool)
    want_card = {}
    for op in OPS:
        got = P.pairwise(op, P, ia, ib).to_wire_list()
        memo = {}
        for p in range(npairs):
            key = (int(ia[p]), int(ib[p]))
            if key not in memo:
                memo[key] = orc.op(op, pool[key[0]], pool[key[1]])
            assert got[p] == memo[key], (op, p)
        cards = P.pairwise_cardinality(op, P, ia, ib).tolist()
        for p in range(npairs):
            key = (op, int(ia[p]), int(ib[p]))
            if key not in want_card:
                want_card[key] = orc.op_cardinality(op, pool[key[1]], pool[key[2]])
            assert cards[p] == want_card[key], (op, p)


def test_device_content_digests_match_oracle(pkg):
    """rs_batch_digests (device) == the oracle's content digest, on the
    reference's golden inputs and on GPU op results of every container mix."""
    g = load()
    ws = [g.wire(a) for a in g["pair_a"]]
    buf = np.frombuffer(b"".join(ws), np.uint8)
    offs = np.concatenate([[0], np.cumsum([len(w) for w in ws])]).astype(np.uint64)
    A = pkg.BitmapBatch.from_wire(ws)
    assert np.array_equal(A.digests(), orc.digest_images(buf, offs))
    B = pkg.BitmapBatch.from_wire([g.wire(b) for b in g["pair_b"]])
    for op in OPS:
        R = A.pairwise(op, B)
        rw = R.to_wire_list()
        rbuf = np.frombuffer(b"".join(rw), np.uint8)
        roffs = np.concatenate([[0], np.cumsum([len(w) for w in rw])]).astype(np.uint64)
        assert np.array_equal(R.digests(), orc.digest_images(rbuf, roffs)), op


def test_all_pairs_direct_rows_variant(pkg, monkeypatch):
    """The experimental direct-row tensor-core tiles (RS_ALLPAIRS_DIRECT=1:
    rows built from the containers -- bitsets, arrays, runs -- inside the
    tile kernel) give the oracle's counts, incl. a 300-container key (block
    tiles with a separate A operand)."""
    rng = np.random.default_rng(78)
    imgs = []
    for i in range(300):
        kind = i % 3
        if kind == 0:
            v = rng.choice(65536, int(rng.integers(1, 4000)), replace=False)
        elif kind == 1:
            v = np.nonzero(rng.random(65536) < rng.uniform(0.1, 0.9))[0]
        else:
            s0 = int(rng.integers(0, 60000))
            v = np.arange(s0, s0 + int(rng.integers(1, 5000)))
        w = orc.from_values(np.asarray(v).astype(np.uint64))
        imgs.append(orc.run_optimize(w)[0] if i % 4 == 0 else w)
    offs = np.zeros(len(imgs) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(x) for x in imgs])
    buf = np.frombuffer(b"".join(imgs), dtype=np.uint8)
    monkeypatch.setenv("RS_ALLPAIRS_DIRECT", "1")
    monkeypatch.setenv("RS_ALLPAIRS_UMMA_MIN", "2")
    _all_pairs_check(pkg, buf, offs)


@pytest.mark.parametrize("radix", ["0", "1"])
def test_union_many_selection_grouping_paths(pkg, monkeypatch, radix):
    """union_many over explicit selections -- repeated and out-of-order
    bitmap indices, and more bitmaps than the counting-sort grouping takes
    (1,100 > 1,024: the radix-sort grouping) -- with both groupings forced,
    against the oracle's sequential fold in selection order."""
    import workloads as synth
    monkeypatch.setenv("RS_GROUP_RADIX", radix)
    buf, offs = synth.config4(nbitmaps=12)
    w = _wires(buf, offs)
    Bt = pkg.BitmapBatch.from_wire((buf, offs))
    for sel in ([3, 1, 3, 0, 11, 1], [5], list(range(11, -1, -1)) * 3):
        assert Bt.union_many(sel).to_wire_list()[0] == orc.union_many([w[i] for i in sel])
    rng = np.random.default_rng(5)
    many = [pkg.RoaringBitmap.from_values(rng.integers(0, 1 << 22, int(rng.integers(0, 300)))).serialize()
            for _ in range(1100)]
    Bm = pkg.BitmapBatch.from_wire(many)
    sel = list(rng.permutation(1100)) + [7, 7]
    assert Bm.union_many(sel).to_wire_list()[0] == orc.union_many([many[i] for i in sel])


@pytest.mark.parametrize("routing", ["3", "1"])
def test_galloping_pair_boundaries(pkg, monkeypatch, routing):
    """array_intersect_galloping's case (kernels/scalar.py:149-176) at the
    edges of its GPU paths: small sides of 1, 31..33, 63..65 and 256 values
    against large sides at exactly 16x, one under, and 4096; the small side on
    either operand; subsets, disjoint and interleaved values; one-container
    pairs (container_pairwise) and the same containers inside bitmaps.  Both
    routings of the short pairs: one warp of the large-pair kernel's group
    (RS_GALLOP_TMA=3, the default) and the galloping kernel (=1)."""
    import subprocess, sys, os, textwrap
    # the routing constant is read once per process: run the body in a child
    code = textwrap.dedent("""
        import numpy as np, sys
        sys.path.insert(0, %r)
        import paper_1709_07821_b200 as pkg
        from oracle import oracle as orc
        rng = np.random.default_rng(64)
        wa, wb = [], []
        for ns in (1, 2, 31, 32, 33, 63, 64, 65, 128, 256):
            for nl in sorted({max(16 * ns - 1, ns + 1), 16 * ns, 16 * ns + 1, 4096}):
                if nl > 4096 or ns + nl <= 256:
                    continue
                for kind in ("subset", "disjoint", "mixed"):
                    L = np.sort(rng.choice(65536, size=nl, replace=False)).astype(np.uint64)
                    if kind == "subset":
                        S = np.sort(rng.choice(L, size=ns, replace=False))
                    elif kind == "disjoint":
                        S = np.sort(rng.choice(np.setdiff1d(np.arange(65536, dtype=np.uint64), L), size=ns, replace=False))
                    else:
                        S = np.unique(np.concatenate([rng.choice(L, size=(ns + 1) // 2, replace=False),
                                                      rng.choice(65536, size=ns, replace=False).astype(np.uint64)]))[:ns]
                    for small_first in (True, False):
                        a, b = (S, L) if small_first else (L, S)
                        wa.append(orc.from_values(a)); wb.append(orc.from_values(b))
        A = pkg.BitmapBatch.from_wire(wa); B = pkg.BitmapBatch.from_wire(wb)
        for op in ("and", "or", "andnot", "xor"):
            want = [orc.op(op, x, y) for x, y in zip(wa, wb)]
            for got in (A.container_pairwise(op, B).to_wire_list(), A.pairwise(op, B).to_wire_list()):
                bad = [i for i in range(len(wa)) if got[i] != want[i]]
                assert not bad, (op, bad[:5])
            wc = [orc.op_cardinality(op, x, y) for x, y in zip(wa, wb)]
            assert A.container_pairwise_cardinality(op, B).tolist() == wc, op
            assert A.pairwise_cardinality(op, B).tolist() == wc, op
        print("pairs", len(wa))
    """) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RS_GALLOP_TMA=routing)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
