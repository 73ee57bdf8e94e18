"""Drop-in edge cases on the GPU: empty and non-canonical containers at the
container level (pinned on golden_v2.npz, produced by the real reference with
tests/golden/make_golden_v2.py), empty images in the batched container path,
result-pool packing, the pinned readback pool's lifetime, and deferred
ingest of malformed arrays staying in bounds."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
OPS = ("and", "or", "andnot", "xor")
GOLDEN2 = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "golden_v2.npz")


@pytest.fixture(scope="module")
def pkg():
    import paper_1709_07821_b200 as p
    return p


def decode(pkg, blob: bytes):
    tag, body = blob[0], blob[1:]
    if tag == 1:
        return pkg.ArrayContainer(np.frombuffer(body, "<u2").astype(np.uint16))
    if tag == 2:
        card = int.from_bytes(body[:4], "little")
        return pkg.BitsetContainer(np.frombuffer(body[4:], "<u8").astype(np.uint64), card)
    return pkg.RunContainer(np.frombuffer(body, "<u2").astype(np.uint16).reshape(-1, 2))


def members(pkg, c):
    from paper_1709_07821_b200.containers import container_positions
    return container_positions(c)


def test_golden_edge_container_pairs(pkg):
    """containers.py:450-570 on empty / under-full / over-full / non-minimal
    containers: result type tag, members and counts equal the reference's."""
    z = np.load(GOLDEN2)
    buf, off = z["cont_buf"], z["cont_off"]
    blobs = [buf[int(off[i]):int(off[i + 1])].tobytes() for i in range(len(off) - 1)]
    kinds = [str(k) for k in z["kinds"]]
    bad = []
    for p, kind in enumerate(kinds):
        a, b = decode(pkg, blobs[2 * p]), decode(pkg, blobs[2 * p + 1])
        for k, op in enumerate(OPS):
            i = 4 * p + k
            want = z["res_members"][int(z["res_off"][i]):int(z["res_off"][i + 1])]
            r = pkg.container_pairwise(op, a, b)
            if r.tag != int(z["res_tag"][i]) or not np.array_equal(members(pkg, r), want):
                bad.append((kind, op, "result", r.tag, int(z["res_tag"][i])))
            c = pkg.container_pairwise_cardinality(op, a, b)
            if c != int(z["counts"][i]):
                bad.append((kind, op, "count", c, int(z["counts"][i])))
    assert not bad, bad[:10]


def test_batched_container_pairs_with_empty_images(pkg):
    """A zero-container image is the empty container in the batched
    container path: OR/XOR keep the other side, ANDNOT keeps A, AND drops."""
    g = __import__("tests.golden_io", fromlist=["load"]).load()
    ws_a = [g.wire(a) for a in g["cont_a"]][:40]
    ws_b = [g.wire(b) for b in g["cont_b"]][:40]
    empty = b"ROAR\x00\x00\x00\x00"
    rng = np.random.default_rng(5)
    ea = rng.random(40) < 0.3
    eb = rng.random(40) < 0.3
    A = pkg.BitmapBatch.from_wire([empty if e else w for e, w in zip(ea, ws_a)])
    B = pkg.BitmapBatch.from_wire([empty if e else w for e, w in zip(eb, ws_b)])
    for k, op in enumerate(OPS):
        got = A.container_pairwise(op, B).to_wire_list()
        cards = A.container_pairwise_cardinality(op, B).tolist()
        for p in range(40):
            if ea[p] or eb[p]:
                keep = (ws_b[p] if not eb[p] and op in ("or", "xor") else None) if ea[p] else \
                    (ws_a[p] if op != "and" else None)
                want = keep if keep is not None else empty
                # container-level results ignore keys: compare count, tag, card, payload
                assert got[p][10:] == want[10:] and got[p][4:8] == want[4:8], (op, p)
                assert cards[p] == (0 if keep is None else int.from_bytes(want[12:16], "little")), (op, p)
            else:  # golden pairs share one key: the reference's container_pairwise result
                assert got[p] == g.wire(g["cont_res"][p][k]), (op, p)
                assert cards[p] == int(g["cont_card"][p][k]), (op, p)


def test_result_pools_are_packed(pkg):
    """Upper-bound result pools are packed when the host looks at them:
    pool bytes <= 1.25x the containers' bytes (config-4 AND and union_many)."""
    import workloads as synth
    nb = 200
    buf, offs = synth.config4(nbitmaps=nb)
    Bt = pkg.BitmapBatch.from_wire((buf, offs))
    ia, ib = np.arange(nb - 1), np.arange(1, nb)
    for R in (Bt.pairwise("and", Bt, ia, ib), Bt.pairwise("or", Bt, ia, ib), Bt.union_many()):
        _, nc, pool = R.info()
        payload, _, types = R.stats()
        padded = payload + 16 * nc  # pool slots are 16-byte aligned
        assert pool <= 1.25 * padded + 4096, (pool, payload, nc)
    R = Bt.pairwise("and", Bt, ia, ib)
    assert R.info()[2] <= 0.15e9


def test_pinned_readback_pool_lifetime(pkg):
    """all_pairs_cardinality results stay valid while the caller holds them
    (the pooled page-locked block returns only when the last view dies)."""
    import workloads as synth
    buf, offs = synth.config5(nbitmaps=128)
    B = pkg.BitmapBatch.from_wire((buf, offs))
    inter1, uni1 = B.all_pairs_cardinality()
    keep = inter1.copy(), uni1.copy()
    X = pkg.BitmapBatch.from_wire((buf, offs)).select(list(range(127, -1, -1)))
    inter2, uni2 = X.all_pairs_cardinality()   # same sizes: would reuse a released block
    assert np.array_equal(inter1, keep[0]) and np.array_equal(uni1, keep[1])
    assert not np.shares_memory(inter1, inter2)


def test_deferred_ingest_of_duplicate_array_stays_in_bounds(pkg):
    """An array payload with repeated values (V_ARRAY_ORDER) read through the
    deferred ingest: ops queued before the check see only the strictly
    increasing prefix, and wait() raises the reference's DecodeError."""
    vals = np.arange(0, 4000, dtype=np.uint16)
    vals[2000:] = 1999  # 2000 copies of one value
    img = bytearray(b"ROAR" + (1).to_bytes(4, "little") + (0).to_bytes(2, "little") + bytes([1, 0])
                    + (4000).to_bytes(4, "little") + vals.astype("<u2").tobytes())
    pin = pkg._lib.PinnedBuffer(len(img))
    pin.array[:] = np.frombuffer(bytes(img), np.uint8)
    D = pkg.BitmapBatch.from_wire((pin.array, np.array([0, len(img)], np.uint64)), deferred=True)
    other = pkg.BitmapBatch.from_values([np.arange(0, 4000, dtype=np.uint32)])
    R = D.pairwise("and", other)          # queued before the checks are read back
    R2 = D.container_pairwise("or", other)
    with pytest.raises(pkg.DecodeError):
        D.wait()
    # results were computed from the 2000-value prefix, nothing past the slots
    assert int(R.cardinalities()[0]) <= 2000
    assert int(R2.cardinalities()[0]) <= 4000


def test_to_wire_async_matches_sync_export(pkg):
    """rs_batch_to_wire_async: same images and offsets as rs_batch_to_wire,
    landing in pinned memory behind a completion event; the result batch may
    be freed before the copy finishes; too small a buffer is an error."""
    from tests.golden_io import load
    g = load()
    A = pkg.BitmapBatch.from_wire([g.wire(a) for a in g["pair_a"]])
    B = pkg.BitmapBatch.from_wire([g.wire(b) for b in g["pair_b"]])
    pin = pkg._lib.PinnedBuffer(64 << 20)
    for op in OPS:
        R = A.pairwise(op, B)
        want_buf, want_offs = R.to_wire()
        offs, done = R.to_wire_async(pin.array)
        del R  # freed while the copy may still be in flight
        done.wait()
        assert done.done()
        assert np.array_equal(offs, want_offs), op
        assert pin.array[:int(offs[-1])].tobytes() == want_buf.tobytes(), op
    R = A.pairwise("or", B)
    with pytest.raises(ValueError):
        R.to_wire_async(np.zeros(16, np.uint8))


def test_from_wire_device_matches_host_ingest(pkg):
    """rs_batch_from_wire_device: images already in HBM, descriptor walk on the
    device -- same batch as the host path on the reference's golden images
    (all container types), and the exact DecodeError on every malformed one."""
    import torch
    from tests.golden_io import load
    g = load()
    ws = [g.wire(a) for a in g["pair_a"]] + [g.wire(b) for b in g["pair_b"]] + [b"ROAR\x00\x00\x00\x00"]
    buf = np.frombuffer(b"".join(ws), np.uint8)
    offs = np.concatenate([[0], np.cumsum([len(w) for w in ws])]).astype(np.uint64)
    dbuf = torch.from_numpy(buf.copy()).cuda()
    doffs = torch.from_numpy(offs.astype(np.int64)).cuda()
    D = pkg.BitmapBatch.from_wire_device(dbuf.data_ptr(), doffs.data_ptr(), len(ws))
    H = pkg.BitmapBatch.from_wire(ws)
    assert D.to_wire_list() == ws
    assert np.array_equal(D.digests(), H.digests())
    assert np.array_equal(D.cardinalities(), H.cardinalities())
    assert D.pairwise("xor", H).to_wire_list() == H.pairwise("xor", H).to_wire_list()
    # malformed images: the host path's exact error (offset and message)
    for bi in g["bad"]:
        img = g.wire(bi)
        with pytest.raises(pkg.DecodeError) as e1:
            pkg.BitmapBatch.from_wire([ws[0], img])
        t = torch.from_numpy(np.frombuffer(ws[0] + img, np.uint8).copy()).cuda()
        o = torch.tensor([0, len(ws[0]), len(ws[0]) + len(img)], dtype=torch.int64).cuda()
        with pytest.raises(pkg.DecodeError) as e2:
            pkg.BitmapBatch.from_wire_device(t.data_ptr(), o.data_ptr(), 2)
        assert str(e1.value) == str(e2.value) and e1.value.offset == e2.value.offset
