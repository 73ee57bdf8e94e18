"""Full-size parity on the five BASELINE.json configs: every result image of
every pair (as a digest) and every count, GPU vs the C oracle on the same
seeded inputs, plus size-independent identities.  Runs in ~1-2 minutes on a
B200 box (the oracle uses all host cores)."""
import hashlib

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu
OPS = ("and", "or", "andnot", "xor")


def digests(buf, offs):
    return [hashlib.blake2b(buf[int(offs[i]):int(offs[i + 1])].tobytes(), digest_size=16).digest()
            for i in range(len(offs) - 1)]


def oracle_digests(op, bufA, offA, bufB, offB, ia, ib, chunk=4096):
    out = []
    for s in range(0, len(ia), chunk):
        ws = orc.op_batch(op, bufA, offA, bufB, offB, ia[s:s + chunk], ib[s:s + chunk])
        out += [hashlib.blake2b(w, digest_size=16).digest() for w in ws]
    return out


def test_config2_full(pkg_full):
    rb, synth = pkg_full
    n = 1024
    buf, offs = synth.config2()
    ia_img, ib_img = synth.slice_images(buf, offs, 0, n), synth.slice_images(buf, offs, n, 2 * n)
    A, B = rb.BitmapBatch.from_wire(ia_img), rb.BitmapBatch.from_wire(ib_img)
    idx = np.arange(n)
    cA, cB = A.cardinalities().astype(np.int64), B.cardinalities().astype(np.int64)
    inter = A.pairwise_cardinality("and", B).astype(np.int64)
    for op in OPS:
        R = A.pairwise(op, B)
        assert digests(*R.to_wire()) == oracle_digests(op, *ia_img, *ib_img, idx, idx), op
        cnt = A.pairwise_cardinality(op, B).astype(np.int64)
        assert np.array_equal(cnt, R.cardinalities().astype(np.int64))
        want = {"and": inter, "or": cA + cB - inter, "andnot": cA - inter, "xor": cA + cB - 2 * inter}[op]
        assert np.array_equal(cnt, want)                       # bitmap.py:235-241 identities


def test_config3_full(pkg_full):
    rb, synth = pkg_full
    n = 1_000_000
    buf, offs = synth.config3(npairs=n)
    ia_img, ib_img = synth.slice_images(buf, offs, 0, n), synth.slice_images(buf, offs, n, 2 * n)
    A, B = rb.BitmapBatch.from_wire(ia_img), rb.BitmapBatch.from_wire(ib_img)
    SA, SB = orc.Session(*ia_img), orc.Session(*ib_img)
    idx = np.arange(n)
    for op in OPS:
        R = A.container_pairwise(op, B)
        assert digests(*R.to_wire()) == oracle_digests(op, *ia_img, *ib_img, idx, idx, chunk=65536), op
        got = A.container_pairwise_cardinality(op, B).astype(np.int64)
        assert np.array_equal(got, SA.run(op, "container_pairwise_cardinality", SB, idx, idx)), op


def test_config4_full(pkg_full):
    rb, synth = pkg_full
    nb = 200
    buf, offs = synth.config4(nbitmaps=nb)
    Bt = rb.BitmapBatch.from_wire((buf, offs))
    ia, ib = np.arange(nb - 1), np.arange(1, nb)
    for op in OPS:
        R = Bt.pairwise(op, Bt, ia, ib)
        assert digests(*R.to_wire()) == oracle_digests(op, buf, offs, buf, offs, ia, ib), op
        S = orc.Session(buf, offs)
        got = Bt.pairwise_cardinality(op, Bt, ia, ib).astype(np.int64)
        assert np.array_equal(got, S.run(op, "op_cardinality", S, ia, ib)), op
    wires = [buf[int(offs[i]):int(offs[i + 1])].tobytes() for i in range(nb)]
    assert Bt.union_many().to_wire_list()[0] == orc.union_many(wires)


def test_config5_full(pkg_full):
    rb, synth = pkg_full
    nb = 512
    buf, offs = synth.config5(nbitmaps=nb)
    Bt = rb.BitmapBatch.from_wire((buf, offs))
    inter, uni = Bt.all_pairs_cardinality()
    pi, pj = np.triu_indices(nb, 1)
    want = orc.all_pairs_and(buf, offs, pi, pj)
    assert np.array_equal(inter.astype(np.int64), want)
    c = Bt.cardinalities().astype(np.int64)
    assert np.array_equal(uni.astype(np.int64), c[pi] + c[pj] - want)


def test_config1_full_and_run_optimize_roundtrip(pkg_full):
    rb, synth = pkg_full
    buf, offs = synth.config1()
    w = [buf[int(offs[i]):int(offs[i + 1])].tobytes() for i in range(2)]
    a, b = rb.RoaringBitmap.deserialize(w[0]), rb.RoaringBitmap.deserialize(w[1])
    for op in OPS:
        assert a.op(op, b).serialize() == orc.op(op, w[0], w[1])
    # from_values on the GPU over the exported values reproduces the images
    V = rb.BitmapBatch.from_values([orc.to_array(x) for x in w])
    assert V.to_wire_list() == w


@pytest.fixture(scope="module")
def pkg_full():
    import paper_1709_07821_b200 as rb
    import workloads as synth
    return rb, synth
