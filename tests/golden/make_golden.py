"""Generate golden vectors by running the REAL reference (roaringset, pure Python).

Run here (the reference is importable only in the build container):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports /root/reference/pkg/src/roaringset read-only and writes
tests/golden/golden_v1.npz.  The fixture pins the C oracle (oracle/) and, via
the oracle, the CUDA path.  Cases:

* ``pair_*``   -- random bitmap pairs of every container mix (arrays, bitsets,
                  runs; run_optimize'd or not): the 4 materialized ops as wire
                  bytes (serde.serialize), and the 4 op_cardinality values.
* ``cont_*``   -- single-container pairs drawn like tests/test_containers.py's
                  any_container strategy (all 9 type pairs) plus
                  container_pairwise_cardinality for all ops.
* ``um_*``     -- union_many over random bitmap lists (order-dependent types,
                  SURVEY App. B) including the [R,X,Y] / [X,Y,R] pin.
* ``fv_*``     -- from_values on unsorted inputs with duplicates, then
                  run_optimize (+ changed flag) and to_array.
* ``bad_*``    -- corrupted wire images with the DecodeError offset/message.
* ``mem_*``    -- membership queries (members, neighbours, misses) per bitmap.
* ``mut_*``    -- add/remove sequences: changed flags and the image after each.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = os.environ.get("ROARINGSET_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import roaringset as rs  # noqa: E402
import roaringset.containers as ct  # noqa: E402
from roaringset import RoaringBitmap, serialize  # noqa: E402

OPS = ("and", "or", "andnot", "xor")
CHUNK = 1 << 16
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")


def chunk_values(rng, key: int, style: str) -> np.ndarray:
    if style == "sparse":
        n = int(rng.integers(1, 600))
        v = rng.integers(0, CHUNK, size=n)
    elif style == "mid":
        n = int(rng.integers(2000, 4200))
        v = rng.integers(0, CHUNK, size=n)
    elif style == "dense":
        n = int(rng.integers(4097, 12000))
        v = rng.integers(0, CHUNK, size=n)
    elif style == "runs":
        v = []
        pos = int(rng.integers(0, 2000))
        while pos < CHUNK:
            ln = int(rng.geometric(1 / 40))
            v.append(np.arange(pos, min(pos + ln, CHUNK)))
            pos += ln + int(rng.geometric(1 / 200))
            if rng.random() < 0.02:
                break
        v = np.concatenate(v) if v else np.array([5])
    elif style == "bigrun":
        s = int(rng.integers(0, 30000))
        v = np.arange(s, min(CHUNK, s + int(rng.integers(1, 35000))))
    elif style == "tie":  # 2 runs over 4 values -> strict tie goes to array
        s = int(rng.integers(0, 60000))
        v = np.array([s, s + 1, s + 10, s + 11])
    else:  # "evens": bitset with many runs
        s = int(rng.integers(0, 20000))
        v = np.arange(s, min(CHUNK, s + 2 * int(rng.integers(4100, 9000))), 2)
    return np.unique(v.astype(np.int64)) + key * CHUNK


STYLES = ("sparse", "mid", "dense", "runs", "bigrun", "tie", "evens")


def random_bitmap(rng, keyspace: int, max_chunks: int = 4) -> RoaringBitmap:
    n = int(rng.integers(0, max_chunks + 1))
    keys = rng.choice(keyspace, size=min(n, keyspace), replace=False)
    parts = [chunk_values(rng, int(k), STYLES[int(rng.integers(0, len(STYLES)))]) for k in keys]
    vals = np.unique(np.concatenate(parts)) if parts else np.array([], dtype=np.int64)
    rb = RoaringBitmap.from_values(vals.astype(np.uint64))
    if rng.random() < 0.6:
        rb.run_optimize()
    return rb


def related(rng, a: RoaringBitmap, keyspace: int) -> RoaringBitmap:
    """Second bitmap of a pair: often shares chunks/values with the first."""
    if len(a) and rng.random() < 0.5:
        av = a.to_array().astype(np.int64)
        keep = av[rng.random(len(av)) < rng.uniform(0.2, 0.9)]
        extra = random_bitmap(rng, keyspace).to_array().astype(np.int64)
        rb = RoaringBitmap.from_values(np.unique(np.concatenate([keep, extra])).astype(np.uint64))
        if rng.random() < 0.6:
            rb.run_optimize()
        return rb
    return random_bitmap(rng, keyspace)


def any_container(rng) -> RoaringBitmap:
    """test_containers.py:30-50 any_container, wrapped at a random key."""
    key = int(rng.integers(0, CHUNK))
    kind = ("array", "run", "bitset")[int(rng.integers(0, 3))]
    if kind == "array":
        vals = np.unique(rng.integers(0, CHUNK, size=int(rng.integers(1, 121))))
        c = ct.ArrayContainer(vals.astype(np.uint16))
    elif kind == "run":
        vals = set()
        for _ in range(int(rng.integers(1, 9))):
            s, ln = int(rng.integers(0, 65401)), int(rng.integers(0, 301))
            vals.update(range(s, min(s + ln, 65535) + 1))
        c = ct.container_normalize(ct.ArrayContainer(np.array(sorted(vals), dtype=np.uint16)),
                                   consider_run=True)
    else:
        start, step = int(rng.integers(0, 40001)), int(rng.integers(1, 4))
        count = int(rng.integers(4097, 6001))
        vals = np.arange(start, start + step * count, step, dtype=np.int64)
        vals = vals[vals <= 65535].astype(np.uint16)
        c = ct.ArrayContainer(vals) if len(vals) <= ct.ARRAY_MAX else ct.bitset_from_positions(vals)
    return RoaringBitmap._from_chunks([key], [c]), key


class Pack:
    """Byte strings -> (buf, offsets) for npz storage."""

    def __init__(self):
        self.items: list[bytes] = []

    def add(self, b: bytes) -> int:
        self.items.append(bytes(b))
        return len(self.items) - 1

    def arrays(self):
        offs = np.zeros(len(self.items) + 1, dtype=np.uint64)
        offs[1:] = np.cumsum([len(x) for x in self.items])
        buf = np.frombuffer(b"".join(self.items), dtype=np.uint8) if self.items else np.zeros(0, np.uint8)
        return buf, offs


def main():
    rng = np.random.default_rng(1709_07821)
    wires = Pack()
    out = {}

    # ---------------------------------------------------------- pairs
    pa, pb, pres, pcard = [], [], [], []
    for t in range(160):
        keyspace = (2, 4, 8, 40)[t % 4]
        a = random_bitmap(rng, keyspace)
        b = related(rng, a, keyspace)
        ia, ib = wires.add(serialize(a)), wires.add(serialize(b))
        pa.append(ia)
        pb.append(ib)
        pres.append([wires.add(serialize(a.op(op, b))) for op in OPS])
        pcard.append([a.op_cardinality(op, b) for op in OPS])
    # known answers: test_bitmap.py:78-95, test_containers.py:160-170
    known = [
        ([1, 3, 5, 7], [1, 2, 3, 4, 6, 7, 8, 9]),
        ([5, 70000, 200000], [5, 200000, 999999]),
        (list(range(5000)), list(range(4000, 9000))),
        (list(range(0, 8000, 2)), list(range(1, 8000, 2))),
        ([1, 2, 3], [CHUNK + 1, 2 * CHUNK + 5]),
    ]
    for x, y in known:
        a, b = RoaringBitmap.from_values(x), RoaringBitmap.from_values(y)
        pa.append(wires.add(serialize(a)))
        pb.append(wires.add(serialize(b)))
        pres.append([wires.add(serialize(a.op(op, b))) for op in OPS])
        pcard.append([a.op_cardinality(op, b) for op in OPS])
    out["pair_a"], out["pair_b"] = np.array(pa), np.array(pb)
    out["pair_res"], out["pair_card"] = np.array(pres), np.array(pcard, dtype=np.int64)

    # ------------------------------------------------- container pairs
    ca, cb, cres, ccard, ctypes_ = [], [], [], [], []
    for _ in range(400):
        a, key = any_container(rng)
        b, _k = any_container(rng)
        # same chunk: move b's single container to a's key
        b = RoaringBitmap._from_chunks([key], [next(iter(b.chunks()))[1]])
        ca.append(wires.add(serialize(a)))
        cb.append(wires.add(serialize(b)))
        (ka, A), (kb, B) = next(iter(a.chunks())), next(iter(b.chunks()))
        res = []
        for op in OPS:
            r = ct.container_pairwise(op, A, B)
            res.append(wires.add(serialize(RoaringBitmap._from_chunks([key], [r])) if len(r)
                                 else serialize(RoaringBitmap())))
        cres.append(res)
        ccard.append([ct.container_pairwise_cardinality(op, A, B) for op in OPS])
        ctypes_.append([A.tag, B.tag])
    out["cont_a"], out["cont_b"] = np.array(ca), np.array(cb)
    out["cont_res"], out["cont_card"] = np.array(cres), np.array(ccard, dtype=np.int64)
    out["cont_tags"] = np.array(ctypes_)

    # ---------------------------------------------------- union_many
    um_members, um_res = [], []
    R = RoaringBitmap._from_chunks([0], [ct.RunContainer(np.array([[0, 999]], dtype=np.uint16))])
    X = RoaringBitmap.from_values(range(2000, 4000, 2))
    Y = RoaringBitmap.from_values(range(2001, 4000, 2))
    lists = [[R, X, Y], [X, Y, R], [X], []]
    for _ in range(24):
        n = int(rng.integers(2, 12))
        keyspace = int(rng.integers(2, 10))
        lists.append([random_bitmap(rng, keyspace) for _ in range(n)])
    for lst in lists:
        um_members.append([wires.add(serialize(x)) for x in lst])
        um_res.append(wires.add(serialize(RoaringBitmap.union_many(lst))))
    out["um_members"] = json.dumps(um_members)
    out["um_res"] = np.array(um_res)

    # --------------------------------------------- from_values & co.
    fv_in = Pack()
    fv_res, fv_opt, fv_changed, fv_arr = [], [], [], []
    for t in range(40):
        rb = random_bitmap(rng, 6)
        vals = rb.to_array().astype(np.uint64)
        dup = rng.choice(vals, size=min(len(vals), 50)) if len(vals) else vals
        mixed = np.concatenate([vals, dup])
        rng.shuffle(mixed)
        fv_in.add(mixed.astype("<u8").tobytes())
        b = RoaringBitmap.from_values(mixed)
        fv_res.append(wires.add(serialize(b)))
        fv_arr.append(wires.add(b.to_array().astype("<u4").tobytes()))
        changed = b.run_optimize()
        fv_opt.append(wires.add(serialize(b)))
        fv_changed.append(int(changed))
    out["fv_in_buf"], out["fv_in_off"] = fv_in.arrays()
    out["fv_res"], out["fv_opt"] = np.array(fv_res), np.array(fv_opt)
    out["fv_changed"], out["fv_arr"] = np.array(fv_changed), np.array(fv_arr)

    # ------------------------------------------------- decode errors
    bad, bad_off, bad_msg = [], [], []

    def add_bad(img: bytes):
        try:
            rs.deserialize(bytes(img))
        except rs.DecodeError as e:
            bad.append(wires.add(bytes(img)))
            bad_off.append(e.offset)
            bad_msg.append(str(e))
            return
        raise AssertionError("expected DecodeError")

    img = bytearray(serialize(RoaringBitmap.from_values([1, 2, 3])))
    img[0] = ord("X")
    add_bad(img)
    add_bad(serialize(RoaringBitmap.from_values(range(5000)))[:100])
    two = bytearray(serialize(RoaringBitmap.from_values([1, CHUNK + 1])))
    two[16:18] = b"\x00\x00"
    add_bad(two)
    img = bytearray(serialize(RoaringBitmap.from_values(range(5000))))
    img[12] ^= 1
    add_bad(img)
    add_bad(serialize(RoaringBitmap.from_values([7])) + b"\x00")
    img = bytearray(serialize(RoaringBitmap.from_values([3, 9])))
    img[16:18], img[18:20] = img[18:20], img[16:18]
    add_bad(img)
    img = bytearray(serialize(RoaringBitmap.from_values([3, 9])))
    img[11] = 1
    add_bad(img)  # nonzero pad
    img = bytearray(serialize(RoaringBitmap.from_values([3, 9])))
    img[10] = 7
    add_bad(img)  # unknown tag
    add_bad(b"RO")
    add_bad(b"ROAR\x01\x00")
    rr = RoaringBitmap.from_values(list(range(100)) + list(range(200, 300)))
    rr.run_optimize()
    img = bytearray(serialize(rr))
    img[18:20] = (150).to_bytes(2, "little")  # second run overlaps first
    add_bad(img)
    img = bytearray(serialize(rr))
    img[16:18] = (0).to_bytes(2, "little")  # empty run container
    add_bad(img)
    img = bytearray(serialize(rr))
    img[24:26] = (65500).to_bytes(2, "little")  # run escapes the chunk
    add_bad(img)
    tie = RoaringBitmap._from_chunks([0], [ct.RunContainer(np.array([[0, 1], [10, 1]], dtype=np.uint16))])
    add_bad(serialize(tie))  # run form not the smallest
    img = bytearray(serialize(RoaringBitmap.from_values(range(100))))
    img[12:16] = (0).to_bytes(4, "little")  # array cardinality out of range
    add_bad(img)
    small_bitset = RoaringBitmap._from_chunks([0], [ct.bitset_from_positions(np.arange(10, dtype=np.uint16))])
    add_bad(serialize(small_bitset))  # bitset with only 10 values
    img = bytearray(serialize(rr))
    img[12:16] = (7).to_bytes(4, "little")
    add_bad(img)  # run cardinality mismatch
    out["bad"], out["bad_off"] = np.array(bad), np.array(bad_off)
    out["bad_msg"] = json.dumps(bad_msg)

    # -------------------------------------- membership and point mutation
    # __contains__ (bitmap.py:99-104) on members, neighbours and misses;
    # add/remove sequences (bitmap.py:106-134) with the changed flags and the
    # wire image after every step.
    mem_bm, mem_q, mem_hit = [], [], []
    mut_start, mut_ops, mut_changed, mut_img = [], [], [], []
    starts = []
    runs = RoaringBitmap._from_chunks([1], [ct.RunContainer(np.array([[0, 99], [101, 99], [300, 99]],
                                                                      dtype=np.uint16))])
    starts.append((runs, [("add", CHUNK + 100), ("add", CHUNK + 200), ("add", CHUNK + 201),
                          ("remove", CHUNK + 150), ("remove", CHUNK + 0), ("remove", CHUNK + 399),
                          ("add", CHUNK + 299), ("remove", CHUNK + 5), ("add", 7), ("remove", 7),
                          ("remove", CHUNK + 7), ("add", (1 << 32) - 1)]))
    full = RoaringBitmap.from_values(range(4096))
    starts.append((full, [("add", 5000), ("remove", 5000), ("remove", 0), ("add", 0), ("add", 70000)]))
    dense = RoaringBitmap.from_values(range(0, 8194, 2))
    starts.append((dense, [("remove", 0), ("remove", 2), ("add", 1), ("remove", 1), ("add", 3)]))
    for _ in range(14):
        keyspace = int(rng.integers(2, 6))
        b = random_bitmap(rng, keyspace)
        vals = b.to_array()
        seq = []
        for _k in range(24):
            r = rng.random()
            if r < 0.35 and len(vals):
                seq.append(("remove", int(rng.choice(vals))))
            elif r < 0.6 and len(vals):
                seq.append(("add", int(rng.choice(vals)) + int(rng.choice([-1, 1]))))
            elif r < 0.8:
                seq.append(("add", int(rng.integers(0, keyspace * CHUNK))))
            else:
                seq.append(("remove", int(rng.integers(0, keyspace * CHUNK))))
        starts.append((b, seq))
    for b, seq in starts:
        vals = b.to_array().astype(np.int64)
        q = np.concatenate([vals[:200], vals[:200] + 1, vals[:200] - 1,
                            rng.integers(0, 8 * CHUNK, size=100)]) if len(vals) else rng.integers(0, CHUNK, 50)
        q = np.clip(q, 0, (1 << 32) - 1).astype(np.uint32)
        mem_bm.append(wires.add(serialize(b)))
        mem_q.append(wires.add(q.astype("<u4").tobytes()))
        mem_hit.append(wires.add(np.array([int(v) in b for v in q.tolist()], dtype=np.uint8).tobytes()))
        cur = b.copy()
        mut_start.append(wires.add(serialize(cur)))
        ch, imgs = [], []
        for kind, v in seq:
            ch.append(int(cur.add(v) if kind == "add" else cur.remove(v)))
            imgs.append(wires.add(serialize(cur)))
        mut_ops.append([[kind, v] for kind, v in seq])
        mut_changed.append(ch)
        mut_img.append(imgs)
    out["mem_bm"], out["mem_q"], out["mem_hit"] = np.array(mem_bm), np.array(mem_q), np.array(mem_hit)
    out["mut_start"] = np.array(mut_start)
    out["mut"] = json.dumps({"ops": mut_ops, "changed": mut_changed, "img": mut_img})

    out["wire_buf"], out["wire_off"] = wires.arrays()
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(wires.items)} images, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
