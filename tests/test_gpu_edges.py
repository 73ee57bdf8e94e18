"""Edge cases across the ABI on the GPU: empty batches and zero pairs, the
largest key (65535) and full chunks, empty results of every op, the async
export of an empty result, device ingest of zero images, key ranges that
select nothing -- each against the oracle or its definition."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu
OPS = ("and", "or", "andnot", "xor")
EMPTY = b"ROAR\x00\x00\x00\x00"


@pytest.fixture(scope="module")
def rb():
    import paper_1709_07821_b200 as p
    return p


def test_zero_pairs_and_empty_batches(rb):
    A = rb.BitmapBatch.from_wire([EMPTY, EMPTY])
    for op in OPS:
        R = A.pairwise(op, A, [], [])
        assert len(R) == 0 and R.to_wire_list() == []
        assert A.pairwise_cardinality(op, A, [], []).tolist() == []
        assert A.pairwise(op, A).to_wire_list() == [EMPTY, EMPTY]
        assert A.pairwise_cardinality(op, A).tolist() == [0, 0]
    assert A.union_many().to_wire_list() == [EMPTY]
    inter, uni = A.all_pairs_cardinality()
    assert inter.tolist() == [0] and uni.tolist() == [0]
    Z = rb.BitmapBatch.from_values([])
    assert len(Z) == 0 and Z.to_wire_list() == []


def test_largest_key_and_full_chunks(rb):
    top = np.arange((65535 << 16), (65535 << 16) + 65536, dtype=np.uint64)   # a full last chunk
    odd = np.arange((65535 << 16) + 1, (65535 << 16) + 65536, 2, dtype=np.uint64)
    a = rb.RoaringBitmap.from_values(top)
    b = rb.RoaringBitmap.from_values(odd)
    a.run_optimize()
    wa, wb = a.serialize(), b.serialize()
    for op in OPS:
        assert a.op(op, b).serialize() == orc.op(op, wa, wb), op
        assert a.op_cardinality(op, b) == orc.op_cardinality(op, wa, wb), op
    assert len(a) == 65536 and (0xFFFFFFFF in a) and (0xFFFEFFFF not in a)


def test_ops_that_empty_everything(rb):
    rng = np.random.default_rng(4)
    v = np.unique(rng.integers(0, 1 << 22, 50000)).astype(np.uint32)
    a = rb.RoaringBitmap.from_values(v)
    assert len(a & rb.RoaringBitmap()) == 0
    assert len(a - a) == 0 and len(a ^ a) == 0
    assert (a - a).serialize() == EMPTY
    R = a._b.pairwise("xor", a._b, [0], [0])
    pin = rb._lib.PinnedBuffer(1 << 12)
    offs, done = R.to_wire_async(pin.array)
    done.wait()
    assert offs.tolist() == [0, 8] and pin.array[:8].tobytes() == EMPTY


def test_device_ingest_of_zero_images_and_empty_images(rb):
    import torch
    o = torch.zeros(1, dtype=torch.int64, device="cuda")
    b = torch.zeros(16, dtype=torch.uint8, device="cuda")
    Z = rb.BitmapBatch.from_wire_device(b.data_ptr(), o.data_ptr(), 0)
    assert len(Z) == 0
    e = torch.from_numpy(np.frombuffer(EMPTY * 3, np.uint8).copy()).cuda()
    o3 = torch.tensor([0, 8, 16, 24], dtype=torch.int64, device="cuda")
    E = rb.BitmapBatch.from_wire_device(e.data_ptr(), o3.data_ptr(), 3)
    assert E.to_wire_list() == [EMPTY] * 3


def test_key_range_selecting_nothing(rb):
    B = rb.BitmapBatch.from_values([np.arange(10, dtype=np.uint32), np.arange(1 << 20, (1 << 20) + 5, dtype=np.uint32)])
    R = B.key_range(100, 200)
    assert R.to_wire_list() == [EMPTY, EMPTY]
    assert R.key_range(0, 65536).to_wire_list() == [EMPTY, EMPTY]
    with pytest.raises(ValueError):
        B.key_range(5, 2)


def test_union_many_with_many_contributors_per_key(rb):
    """Keys with more contributors than one metadata window of the union
    kernels: 300 bitmaps sharing key 0 as arrays / runs only (the fold, past
    its 256-contributor window) and key 1 with bitsets among them (the
    order-free OR, several 64-contributor windows)."""
    rng = np.random.default_rng(21)
    imgs = []
    for i in range(300):
        k0 = np.unique(rng.integers(0, 65536, int(rng.integers(1, 300))))
        if i % 3 == 0:
            s = int(rng.integers(0, 60000))
            k0 = np.arange(s, s + int(rng.integers(50, 3000)))  # run-like
        k1 = np.nonzero(rng.random(65536) < 0.2)[0] if i % 7 == 0 else np.unique(rng.integers(0, 65536, 500))
        w = orc.from_values(np.concatenate([k0, 65536 + k1]).astype(np.uint64))
        imgs.append(orc.run_optimize(w)[0] if i % 2 == 0 else w)
    B = rb.BitmapBatch.from_wire(imgs)
    assert B.union_many().to_wire_list()[0] == orc.union_many(imgs)
