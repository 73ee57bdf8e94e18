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
import types

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
    __slots__ = ("values", "capacity")
    tag = TAG_ARRAY

    def __init__(self, values=(), capacity: int = 0):
        self.values = np.asarray(values, dtype=np.uint16)
        self.capacity = max(len(self.values), capacity)

    def __len__(self) -> int:
        return len(self.values)

    def __eq__(self, other) -> bool:
        return isinstance(other, ArrayContainer) and np.array_equal(self.values, other.values)

    def __repr__(self) -> str:
        return f"ArrayContainer(card={len(self)})"

    def copy(self) -> "ArrayContainer":
        return ArrayContainer(self.values.copy(), self.capacity)


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
    __slots__ = ("runs", "capacity")
    tag = TAG_RUN

    def __init__(self, runs, capacity: int = 0):
        self.runs = np.asarray(runs, dtype=np.uint16).reshape(-1, 2)
        self.capacity = max(len(self.runs), capacity)

    def __len__(self) -> int:
        return len(self.runs) + int(self.runs[:, 1].sum(dtype=np.int64))

    def __eq__(self, other) -> bool:
        return isinstance(other, RunContainer) and np.array_equal(self.runs, other.runs)

    def __repr__(self) -> str:
        return f"RunContainer(runs={len(self.runs)}, card={len(self)})"

    def copy(self) -> "RunContainer":
        return RunContainer(self.runs.copy(), self.capacity)


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


def empty_container() -> ArrayContainer:
    """containers.py:106-107."""
    return ArrayContainer()


def bitset_from_positions(positions) -> BitsetContainer:
    """A BitsetContainer holding `positions` (containers.py:113-119).  Host
    value construction (numpy), like the container classes themselves."""
    pos = np.asarray(positions, dtype=np.int64)
    bits = np.zeros(1 << 16, dtype=bool)
    bits[pos] = True
    words = np.frombuffer(np.packbits(bits, bitorder="little").tobytes(), dtype="<u8").astype(np.uint64)
    return BitsetContainer(words, len(pos))


# Names the reference's tests reach through ``containers.kernels`` (its kernel
# backend module, kernels/_shared.py:8-20).  This build has no per-container
# kernel seam; only the shared constants are provided.
kernels = types.SimpleNamespace(OPS=OPS, BLOCK_WORDS=1024, GALLOP_RATIO=64)


def _tag(c) -> int:
    t = getattr(c, "tag", None)
    if t not in (TAG_ARRAY, TAG_BITSET, TAG_RUN):
        raise TypeError(f"unsupported container {type(c)}")
    return t


def _canonical(c: Container) -> bool:
    """Non-empty and in the form container_normalize would keep (the form the
    wire decoder accepts, serde.py:122-164)."""
    n = len(c)
    t = _tag(c)
    if t == TAG_ARRAY:
        return 1 <= n <= ARRAY_MAX and (n < 2 or bool(np.all(np.diff(c.values.astype(np.int64)) > 0)))
    if t == TAG_BITSET:
        return n > ARRAY_MAX
    nr = len(c.runs)
    if nr == 0:
        return False
    r = c.runs.astype(np.int64)
    e = r[:, 0] + r[:, 1]
    if np.any(e > 0xFFFF) or (nr > 1 and np.any(r[1:, 0] <= e[:-1] + 1)):
        return False
    return nr <= RUN_MAX_RUNS if n > ARRAY_MAX else 2 * nr < n


# Result type of container_pairwise per declared input types (SURVEY App. A,
# containers.py:459-527): "card" = array iff card <= 4096 else bitset
# (_container_from_values / _container_from_words); "run" = container_normalize
# of the interval result (run iff admissible, else by card); "array" = a subset
# of the array side, kept as an ArrayContainer whatever its size.
def _result_rule(ta: int, tb: int, op: str) -> str:
    if ta == tb and ta != TAG_RUN:
        return "card"
    if {ta, tb} == {TAG_ARRAY, TAG_BITSET}:
        if op == "and" or (op == "andnot" and ta == TAG_ARRAY):
            return "array"
        return "card"
    if ta == tb == TAG_RUN:
        return "run"
    if ta == TAG_RUN and tb == TAG_ARRAY:
        return "array" if op == "and" else "run"
    if ta == TAG_ARRAY and tb == TAG_RUN:
        return "array" if op in ("and", "andnot") else "run"
    return "card"


def _device_single(c: Container):
    """One-container device batch holding c's members in canonical form; None
    when c is empty.  Canonical containers go up as wire images; others (an
    under-full bitset, an array over 4096 values, a run form that is not the
    smallest) are rebuilt from their members (from_values on the GPU)."""
    from .batch import BitmapBatch
    if len(c) == 0:
        return None
    if _canonical(c):
        return BitmapBatch.from_wire([_single(c)])
    return BitmapBatch.from_values([container_positions(c).astype(np.uint32)])


def _retype(R, rule: str) -> Container:
    """The one-container device result R re-typed by `rule` (see
    _result_rule); the conversions run on the GPU."""
    from .batch import BitmapBatch
    if R is None or int(R.container_counts()[0]) == 0:
        return ArrayContainer()
    if rule == "array":
        return ArrayContainer(R.to_arrays()[0].astype(np.uint16))
    _, conts = chunks_from_wire(R.to_wire_list()[0])
    if rule == "run":
        R = R.select([0])
        R.run_optimize()                    # run iff admissible, else by card
    elif isinstance(conts[0], RunContainer):  # "card": drop the run form
        R = BitmapBatch.from_values([R.to_arrays()[0]])
    else:
        return conts[0]
    _, conts = chunks_from_wire(R.to_wire_list()[0])
    return conts[0]


def container_pairwise(op: str, a: Container, b: Container) -> Container:
    """containers.py:450-529 on the GPU; an empty result is an empty
    ArrayContainer.  Canonical non-empty inputs run as one batched container
    op whose kernels pick the reference's result type directly.  Empty or
    non-canonical inputs (accepted by the reference as structurally valid
    containers) run on their canonical device forms and the result is
    re-typed by the declared input types' rule (_result_rule), so the type
    matches the reference's dispatch on the objects actually passed."""
    op_index(op)
    ta, tb = _tag(a), _tag(b)
    if _canonical(a) and _canonical(b):
        from .batch import BitmapBatch
        A = BitmapBatch.from_wire([_single(a)])
        B = BitmapBatch.from_wire([_single(b)])
        R = A.container_pairwise(op, B)
        keys, conts = chunks_from_wire(R.to_wire_list()[0])
        return conts[0] if conts else ArrayContainer()
    A, B = _device_single(a), _device_single(b)
    if A is None or B is None:
        # op(empty, x) = x for OR/XOR; op(x, empty) = x for OR/XOR/ANDNOT
        R = (B if op in ("or", "xor") else None) if A is None else (A if op != "and" else None)
    else:
        R = A.container_pairwise(op, B)
    return _retype(R, _result_rule(ta, tb, op))


def container_pairwise_cardinality(op: str, a: Container, b: Container) -> int:
    """containers.py:554-570 on the GPU.  Empty containers count as 0 members
    (|a op empty| from the reference's own formula, containers.py:563-570)."""
    op_index(op)
    _tag(a), _tag(b)
    A, B = _device_single(a), _device_single(b)
    if A is None or B is None:
        la, lb = len(a), len(b)
        return {"and": 0, "or": la + lb, "andnot": la, "xor": la + lb}[op]
    return int(A.container_pairwise_cardinality(op, B)[0])


# ------------------------------------------------- single-container helpers
# The reference's element-level container functions (containers.py:208-367),
# for drop-in completeness.  Each runs as a one-container GPU batch; the
# batched forms are BitmapBatch.contains / pairwise.

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


def container_validate(c: Container, normalized: bool = True) -> None:
    """Raise AssertionError if a host container breaks its invariants
    (containers.py:575-604): the same checks the wire decoder applies."""
    t = _tag(c)
    if t == TAG_ARRAY:
        assert c.values.dtype == np.uint16
        assert len(c.values) <= ARRAY_MAX, "array container over 4096 values"
        if len(c.values) > 1:
            assert np.all(np.diff(c.values.astype(np.int32)) > 0), "array values not strictly increasing"
        assert getattr(c, "capacity", len(c.values)) >= len(c.values)
        return
    if t == TAG_BITSET:
        assert c.words.dtype == np.uint64 and len(c.words) == 1024
        true_card = int(np.bitwise_count(c.words).sum(dtype=np.int64))
        assert c.cardinality == true_card, f"bitset cardinality {c.cardinality} != popcount {true_card}"
        if normalized:
            assert c.cardinality > ARRAY_MAX, "bitset container under 4097 values"
        return
    assert c.runs.dtype == np.uint16 and c.runs.ndim == 2 and c.runs.shape[1] == 2
    runs = c.runs.astype(np.int32)
    assert len(runs) > 0, "empty run container"
    ends = runs[:, 0] + runs[:, 1]
    assert np.all(ends <= 65535)
    if len(runs) > 1:
        assert np.all(runs[1:, 0] > ends[:-1] + 1), "runs overlap or are adjacent"
    if normalized:
        n = len(c)
        assert (len(runs) <= RUN_MAX_RUNS if n > ARRAY_MAX else 2 * len(runs) < n), "run form not the smallest"
