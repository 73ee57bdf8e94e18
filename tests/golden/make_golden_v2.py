"""Golden vectors, part 2: container-level edge cases, from the REAL reference.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_v2.py

Imports /root/reference/pkg/src/roaringset read-only and writes
tests/golden/golden_v2.npz: container pairs where a side is EMPTY (array,
run or bitset form) or NOT CANONICAL (a bitset holding <= 4096 values, an
array holding > 4096, a run form that is not the smallest), which the
reference's container_pairwise / container_pairwise_cardinality accept
(containers.py:450-570; its own strategies draw empty containers,
tests/test_containers.py:24-50).  For each pair and op: the result's type
tag and members, and the count.

Encoding of one container: tag u8 | payload (array: u16 values; bitset:
u32 stored cardinality + 1024 x u64 words; run: u16 (start, length) pairs).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("ROARINGSET_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import roaringset.containers as ct  # noqa: E402

OPS = ("and", "or", "andnot", "xor")
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v2.npz")


def enc(c) -> bytes:
    if isinstance(c, ct.ArrayContainer):
        return bytes([1]) + c.values.astype("<u2").tobytes()
    if isinstance(c, ct.BitsetContainer):
        return bytes([2]) + int(c.cardinality).to_bytes(4, "little") + c.words.astype("<u8").tobytes()
    return bytes([3]) + c.runs.astype("<u2").tobytes()


def runs_of(values: np.ndarray) -> np.ndarray:
    return ct._runs_from_positions(np.asarray(values, dtype=np.uint16))


def make(rng, kind: str):
    if kind == "empty_array":
        return ct.ArrayContainer()
    if kind == "empty_run":
        return ct.RunContainer(np.empty((0, 2), dtype=np.uint16))
    if kind == "empty_bitset":
        return ct.BitsetContainer(np.zeros(1024, dtype=np.uint64), 0)
    if kind == "small_bitset":       # bitset form of 1..4096 values
        n = int(rng.integers(1, 4097))
        return ct.bitset_from_positions(np.sort(rng.choice(65536, n, replace=False)).astype(np.uint16))
    if kind == "big_array":          # array form of 4097..9000 values
        n = int(rng.integers(4097, 9001))
        return ct.ArrayContainer(np.sort(rng.choice(65536, n, replace=False)).astype(np.uint16))
    if kind == "tie_run":            # 2 runs over 4 values: not strictly smaller
        s = int(rng.integers(0, 60000))
        return ct.RunContainer(np.array([[s, 1], [s + 10, 1]], dtype=np.uint16))
    if kind == "single_runs":        # many length-0 runs: run form of a sparse set
        v = np.sort(rng.choice(np.arange(0, 65536, 2), int(rng.integers(2, 3000)), replace=False))
        return ct.RunContainer(runs_of(v))
    if kind == "many_runs":          # > 2047 runs holding > 4096 values
        starts = np.arange(0, 65536, 24)[:int(rng.integers(2100, 2700))]
        return ct.RunContainer(np.stack([starts, np.full_like(starts, 2)], axis=1).astype(np.uint16))
    # canonical containers of each type
    if kind == "array":
        n = int(rng.integers(1, 4097))
        return ct.ArrayContainer(np.sort(rng.choice(65536, n, replace=False)).astype(np.uint16))
    if kind == "bitset":
        n = int(rng.integers(4097, 30000))
        return ct.bitset_from_positions(np.sort(rng.choice(65536, n, replace=False)).astype(np.uint16))
    # "run": a few long intervals
    v = []
    pos = int(rng.integers(0, 3000))
    for _ in range(int(rng.integers(1, 12))):
        ln = int(rng.integers(1, 3000))
        v.append(np.arange(pos, min(pos + ln, 65536)))
        pos += ln + int(rng.integers(2, 4000))
        if pos >= 65536:
            break
    return ct.container_normalize(ct.ArrayContainer(np.unique(np.concatenate(v)).astype(np.uint16)),
                                  consider_run=True)


EDGE = ("empty_array", "empty_run", "empty_bitset", "small_bitset", "big_array", "tie_run", "single_runs",
        "many_runs")
CANON = ("array", "bitset", "run")


def main():
    rng = np.random.default_rng(20261020)
    blobs, kinds, res_tag, res_members, counts = [], [], [], [], []
    pairs = [(x, y) for x in EDGE + CANON for y in EDGE + CANON if x in EDGE or y in EDGE]
    for ka, kb in pairs:
        a, b = make(rng, ka), make(rng, kb)
        blobs += [enc(a), enc(b)]
        kinds.append(f"{ka}|{kb}")
        for op in OPS:
            r = ct.container_pairwise(op, a, b)
            res_tag.append(r.tag)
            res_members.append(ct.container_positions(r).astype(np.uint16))
            counts.append(ct.container_pairwise_cardinality(op, a, b))
            assert counts[-1] == len(r)
    off = np.zeros(len(blobs) + 1, dtype=np.uint64)
    np.cumsum([len(x) for x in blobs], out=off[1:])
    moff = np.zeros(len(res_members) + 1, dtype=np.uint64)
    np.cumsum([len(x) for x in res_members], out=moff[1:])
    np.savez_compressed(OUT, cont_buf=np.frombuffer(b"".join(blobs), dtype=np.uint8), cont_off=off,
                        kinds=np.array(kinds), res_tag=np.array(res_tag, dtype=np.uint8),
                        res_members=np.concatenate(res_members), res_off=moff,
                        counts=np.array(counts, dtype=np.int64))
    print(f"wrote {OUT}: {len(kinds)} container pairs x 4 ops")


if __name__ == "__main__":
    main()
