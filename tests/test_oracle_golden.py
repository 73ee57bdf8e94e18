"""Pin the C oracle (oracle/roaring_oracle.c) against golden vectors produced by
the real reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.golden_io import load

OPS = ("and", "or", "andnot", "xor")


def test_pairs_materialized_and_counts():
    g = load()
    for a, b, res, card in zip(g["pair_a"], g["pair_b"], g["pair_res"], g["pair_card"]):
        wa, wb = g.wire(a), g.wire(b)
        for k, op in enumerate(OPS):
            assert orc.op(op, wa, wb) == g.wire(res[k]), op
            assert orc.op_cardinality(op, wa, wb) == card[k], op


def test_container_pairs_all_type_combinations():
    g = load()
    seen = set()
    for a, b, res, card, tags in zip(g["cont_a"], g["cont_b"], g["cont_res"], g["cont_card"],
                                     g["cont_tags"]):
        wa, wb = g.wire(a), g.wire(b)
        seen.add(tuple(tags))
        for k, op in enumerate(OPS):
            assert orc.op(op, wa, wb) == g.wire(res[k]), (op, tags)
            assert orc.container_pairwise_cardinality(op, wa, wb) == card[k], (op, tags)
    assert len(seen) == 9  # every container-type pair is pinned


def test_union_many():
    g = load()
    for members, res in zip(g["um_members"], g["um_res"]):
        assert orc.union_many([g.wire(m) for m in members]) == g.wire(res)


def test_union_many_order_dependent_types():
    g = load()
    rxy, xyr = g["um_res"][0], g["um_res"][1]
    # same set, different container types
    assert orc.to_array(g.wire(rxy)).tolist() == orc.to_array(g.wire(xyr)).tolist()
    assert g.wire(rxy) != g.wire(xyr)


def test_from_values_run_optimize_to_array():
    g = load()
    buf, off = g["fv_in_buf"], g["fv_in_off"]
    for i, (res, opt, ch, arr) in enumerate(zip(g["fv_res"], g["fv_opt"], g["fv_changed"],
                                                g["fv_arr"])):
        vals = np.frombuffer(buf[int(off[i]):int(off[i + 1])].tobytes(), dtype="<u8")
        w = orc.from_values(vals)
        assert w == g.wire(res)
        o, changed = orc.run_optimize(w)
        assert o == g.wire(opt) and changed == bool(ch)
        assert orc.to_array(w).tobytes() == g.wire(arr)


def test_from_values_rejects_over_32_bits():
    with pytest.raises(ValueError):
        orc.from_values([1, 1 << 32])


def test_decode_errors_match_reference():
    g = load()
    for img, off, msg in zip(g["bad"], g["bad_off"], g["bad_msg"]):
        with pytest.raises(orc.OracleDecodeError) as e:
            orc.check(g.wire(img))
        assert e.value.offset == off
        assert str(e.value) == msg


def test_roundtrip_every_golden_image():
    g = load()
    bad = set(int(i) for i in g["bad"])
    for i in range(len(g.off) - 1):
        if i in bad:
            continue
        w = g.wire(i)
        if w[:4] != b"ROAR":
            continue  # raw value/array payloads
        assert orc.roundtrip(w) == w


def test_batch_entry_points_agree_with_single():
    g = load()
    wa = [g.wire(a) for a in g["pair_a"]]
    wb = [g.wire(b) for b in g["pair_b"]]
    bufA, offA = orc.concat(wa)
    bufB, offB = orc.concat(wb)
    idx = np.arange(len(wa))
    for k, op in enumerate(OPS):
        outs = orc.op_batch(op, bufA, offA, bufB, offB, idx, idx)
        assert outs == [g.wire(r[k]) for r in g["pair_res"]]
        cards = orc.op_cardinality_batch(op, bufA, offA, bufB, offB, idx, idx)
        assert cards.tolist() == [int(c[k]) for c in g["pair_card"]]


def test_membership_fixture_matches_oracle_export():
    g = load()
    for bm, q, hit in zip(g["mem_bm"], g["mem_q"], g["mem_hit"]):
        vals = orc.to_array(g.wire(bm))
        qs = np.frombuffer(g.wire(q), dtype="<u4")
        want = np.frombuffer(g.wire(hit), dtype=np.uint8).astype(bool)
        assert np.array_equal(np.isin(qs, vals), want)


def test_point_mutation_is_op_with_singleton():
    """add(v) / remove(v) (bitmap.py:106-134) re-type containers exactly like
    OR / ANDNOT with the one-value bitmap {v}: the identity the GPU mirror's
    add/remove rely on, pinned on the reference's own mutation sequences."""
    g = load()
    m = g["mut"]
    for start, ops, changed, imgs in zip(g["mut_start"], m["ops"], m["changed"], m["img"]):
        cur = g.wire(start)
        for (kind, v), ch, img in zip(ops, changed, imgs):
            present = v in set(orc.to_array(cur).tolist())
            assert ch == int(present != (kind == "add")), (kind, v)
            if ch:
                one = orc.from_values(np.array([v], dtype=np.uint64))
                cur = orc.op("or" if kind == "add" else "andnot", cur, one)
            assert cur == g.wire(img), (kind, v)


def _mix(z):
    m = (1 << 64) - 1
    z ^= z >> 30; z = (z * 0xBF58476D1CE4E5B9) & m
    z ^= z >> 27; z = (z * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def digest_py(wire: bytes) -> int:
    """Plain-Python restatement of the content digest (roaring_oracle.c
    "content digests", rs_batch_digests)."""
    import struct
    m = (1 << 64) - 1
    (count,) = struct.unpack_from("<I", wire, 4)
    off = 8 + 8 * count
    d = 0
    for j in range(count):
        key, tag, _pad, card = struct.unpack_from("<HBBI", wire, 8 + 8 * j)
        h = _mix((key << 48) | (tag << 40) | card)
        if tag == 1:
            for i, v in enumerate(struct.unpack_from(f"<{card}H", wire, off)):
                h += _mix((((i << 16) | v) + 0x243F6A8885A308D3) & m)
            off += 2 * card
        elif tag == 2:
            for w, x in enumerate(struct.unpack_from("<1024Q", wire, off)):
                h += _mix((x + w * 0x13198A2E03707344) & m)
            off += 8192
        else:
            (nr,) = struct.unpack_from("<H", wire, off)
            r = struct.unpack_from(f"<{2 * nr}H", wire, off + 2)
            for k in range(nr):
                h += _mix((((k << 32) | (r[2 * k] << 16) | r[2 * k + 1]) + 0xA4093822299F31D0) & m)
            off += 2 + 4 * nr
        d += _mix(((h & m) + (j + 1) * 0x082EFA98EC4E6C89) & m)
    return d & m


def test_content_digest_definition():
    """The oracle's content digest equals its plain-Python restatement on the
    reference's own images (all three container types)."""
    g = load()
    ws = [g.wire(i) for i in list(g["pair_a"][:12]) + list(g["pair_res"][:6, 1])]
    buf = np.frombuffer(b"".join(ws), np.uint8)
    offs = np.concatenate([[0], np.cumsum([len(w) for w in ws])]).astype(np.uint64)
    got = orc.digest_images(buf, offs)
    assert [int(x) for x in got] == [digest_py(w) for w in ws]
    assert len(set(int(x) for x in got)) == len(set(ws))
