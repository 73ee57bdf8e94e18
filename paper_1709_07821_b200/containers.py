"""Host-side container values and the container-level API.

The three container shapes mirror the reference classes
(/root/reference/pkg/src/roaringset/containers.py:38-101): they are what
``RoaringBitmap.chunks()`` hands back for inspection.  The container-level
operations ``container_pairwise`` / ``container_pairwise_cardinality``
(containers.py:450-570) run on the GPU: single calls wrap the two containers
as one-container batches; ``ContainerBatch`` runs millions of pairs per launch.
"""

from __future__ import annotations

import struct

import numpy as np

ARRAY_MAX = 4096          # containers.py:27
RUN_MAX_RUNS = 2047       # containers.py:28
TAG_ARRAY, TAG_BITSET, TAG_RUN = 1, 2, 3   # containers.py:31-33
OPS = ("and", "or", "andnot", "xor")       # kernels/_shared.py:8


def op_index(op: str) -> int:
    if op not in OPS:
        raise ValueError(f"unknown op {op!r}")
    return OPS.index(op)


class ArrayContainer:
    __slots__ = ("values",)
    tag = TAG_ARRAY

    def __init__(self, values=()):
        self.values = np.asarray(values, dtype=np.uint16)

    def __len__(self) -> int:
        return len(self.values)

    def __eq__(self, other) -> bool:
        return isinstance(other, ArrayContainer) and np.array_equal(self.values, other.values)

    def __repr__(self) -> str:
        return f"ArrayContainer(card={len(self)})"

    def copy(self) -> "ArrayContainer":
        return ArrayContainer(self.values.copy())


class BitsetContainer:
    __slots__ = ("words", "cardinality")
    tag = TAG_BITSET

    def __init__(self, words: np.ndarray, cardinality: int):
        self.words = np.asarray(words, dtype=np.uint64)
        self.cardinality = int(cardinality)

    def __len__(self) -> int:
        return self.cardinality

    def __eq__(self, other) -> bool:
        return isinstance(other, BitsetContainer) and np.array_equal(self.words, other.words)

    def __repr__(self) -> str:
        return f"BitsetContainer(card={self.cardinality})"

    def copy(self) -> "BitsetContainer":
        return BitsetContainer(self.words.copy(), self.cardinality)


class RunContainer:
    __slots__ = ("runs",)
    tag = TAG_RUN

    def __init__(self, runs):
        self.runs = np.asarray(runs, dtype=np.uint16).reshape(-1, 2)

    def __len__(self) -> int:
        return len(self.runs) + int(self.runs[:, 1].sum(dtype=np.int64))

    def __eq__(self, other) -> bool:
        return isinstance(other, RunContainer) and np.array_equal(self.runs, other.runs)

    def __repr__(self) -> str:
        return f"RunContainer(runs={len(self.runs)}, card={len(self)})"

    def copy(self) -> "RunContainer":
        return RunContainer(self.runs.copy())


Container = ArrayContainer | BitsetContainer | RunContainer


def container_positions(c: Container) -> np.ndarray:
    """Members of a host container as sorted uint16 (containers.py:158-164)."""
    if isinstance(c, ArrayContainer):
        return c.values
    if isinstance(c, BitsetContainer):
        bits = np.unpackbits(c.words.astype("<u8").view(np.uint8), bitorder="little")
        return np.flatnonzero(bits).astype(np.uint16)
    if len(c.runs) == 0:
        return np.empty(0, dtype=np.uint16)
    return np.concatenate([np.arange(int(s), int(s) + int(l) + 1) for s, l in c.runs.tolist()]).astype(np.uint16)


# ------------------------------------------------------------ wire marshaling

def wire_from_chunks(keys, conts) -> bytes:
    """Wire image (serde.py:3-10) of (key, container) pairs, in key order."""
    out = bytearray(b"ROAR")
    out += struct.pack("<I", len(keys))
    for k, c in zip(keys, conts):
        out += struct.pack("<HBBI", int(k), c.tag, 0, len(c))
    for c in conts:
        if isinstance(c, ArrayContainer):
            out += c.values.astype("<u2").tobytes()
        elif isinstance(c, BitsetContainer):
            out += c.words.astype("<u8").tobytes()
        else:
            out += struct.pack("<H", len(c.runs)) + c.runs.astype("<u2").tobytes()
    return bytes(out)


def chunks_from_wire(data: bytes):
    """Parse a wire image produced by this library into (keys, containers)."""
    (count,) = struct.unpack_from("<I", data, 4)
    keys, conts = [], []
    off = 8 + 8 * count
    for i in range(count):
        key, tag, _pad, card = struct.unpack_from("<HBBI", data, 8 + 8 * i)
        if tag == TAG_ARRAY:
            c = ArrayContainer(np.frombuffer(data, "<u2", card, off).astype(np.uint16))
            off += 2 * card
        elif tag == TAG_BITSET:
            c = BitsetContainer(np.frombuffer(data, "<u8", 1024, off).astype(np.uint64), card)
            off += 8192
        else:
            (nr,) = struct.unpack_from("<H", data, off)
            c = RunContainer(np.frombuffer(data, "<u2", 2 * nr, off + 2).astype(np.uint16))
            off += 2 + 4 * nr
        keys.append(key)
        conts.append(c)
    return keys, conts


def _single(c: Container) -> bytes:
    return wire_from_chunks([0], [c]) if len(c) else wire_from_chunks([], [])


def container_pairwise(op: str, a: Container, b: Container) -> Container:
    """containers.py:450-529 on the GPU; an empty result is an empty ArrayContainer."""
    op_index(op)
    if len(a) == 0 or len(b) == 0:
        raise TypeError("containers must be non-empty (normalized)")
    from .batch import BitmapBatch
    A = BitmapBatch.from_wire([_single(a)])
    B = BitmapBatch.from_wire([_single(b)])
    R = A.container_pairwise(op, B)
    keys, conts = chunks_from_wire(R.to_wire_list()[0])
    return conts[0] if conts else ArrayContainer()


def container_pairwise_cardinality(op: str, a: Container, b: Container) -> int:
    """containers.py:554-570 on the GPU."""
    op_index(op)
    from .batch import BitmapBatch
    A = BitmapBatch.from_wire([_single(a)])
    B = BitmapBatch.from_wire([_single(b)])
    return int(A.container_pairwise_cardinality(op, B)[0])


# ------------------------------------------------- single-container helpers
# The reference's element-level container functions (containers.py:208-367),
# for drop-in completeness.  Each runs as a one-container GPU batch; the
# batched forms are BitmapBatch.contains / pairwise.

def _canonical(c: Container) -> bool:
    n = len(c)
    if isinstance(c, ArrayContainer):
        return 1 <= n <= ARRAY_MAX and bool(np.all(np.diff(c.values.astype(np.int64)) > 0))
    if isinstance(c, BitsetContainer):
        return n > ARRAY_MAX
    nr = len(c.runs)
    return nr > 0 and (nr <= RUN_MAX_RUNS if n > ARRAY_MAX else 2 * nr < n)


def _batch_of(c: Container):
    from .batch import BitmapBatch
    if _canonical(c):
        return BitmapBatch.from_wire([_single(c)])
    return BitmapBatch.from_values([container_positions(c).astype(np.uint32)])


def container_normalize(c: Container, consider_run: bool = False) -> Container:
    """containers.py:208-241: the canonical form; `c` itself when unchanged.
    Run candidacy applies to run inputs always and to others on request."""
    from .batch import BitmapBatch
    if len(c) == 0:
        return c if isinstance(c, ArrayContainer) else ArrayContainer()
    B = BitmapBatch.from_values([container_positions(c).astype(np.uint32)])
    if consider_run or isinstance(c, RunContainer):
        B.run_optimize()
    _, conts = chunks_from_wire(B.to_wire_list()[0])
    n = conts[0]
    return c if type(n) is type(c) and n == c else n


def container_contains(c: Container, v: int) -> bool:
    """containers.py:258-268."""
    if len(c) == 0 or not 0 <= int(v) <= 0xFFFF:
        return False
    return bool(_batch_of(c).contains([int(v)])[0])


def container_add(c: Container, v: int):
    """containers.py:271-319: (container, changed); the re-typing is the OR
    rule with {v} (array full -> bitset, runs re-checked)."""
    if container_contains(c, v):
        return c, False
    one = ArrayContainer(np.array([int(v)], dtype=np.uint16))
    if len(c) == 0:
        return one, True
    return container_pairwise("or", container_normalize(c) if not _canonical(c) else c, one), True


def container_remove(c: Container, v: int):
    """containers.py:322-367: (container, changed); the re-typing is the
    ANDNOT rule with {v} (bitset at 4096 -> array, runs re-checked)."""
    if not container_contains(c, v):
        return c, False
    one = ArrayContainer(np.array([int(v)], dtype=np.uint16))
    return container_pairwise("andnot", container_normalize(c) if not _canonical(c) else c, one), True
