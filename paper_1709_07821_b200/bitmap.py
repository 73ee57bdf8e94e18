"""RoaringBitmap: drop-in for the reference's user-facing class
(/root/reference/pkg/src/roaringset/bitmap.py:29-363), backed by the GPU.

Each instance owns a one-bitmap BitmapBatch in HBM.  Set algebra, counts, wide
unions, exports and run_optimize run as sm_100a kernels through the C ABI;
inputs are never mutated (bitmap.py:8-9).  Container types follow the
reference exactly, so wire images compare byte for byte.
"""

from __future__ import annotations

from typing import Callable, Iterable, Iterator

import numpy as np

from .batch import BitmapBatch
from .containers import OPS, Container, chunks_from_wire, op_index
from ._lib import DecodeError

_EMPTY = b"ROAR\x00\x00\x00\x00"


class RoaringBitmap:
    """Compressed set of 32-bit unsigned integers (GPU-resident)."""

    __slots__ = ("_b", "_snap")

    def __init__(self) -> None:
        self._b = BitmapBatch.from_wire([_EMPTY])
        self._snap = None

    @classmethod
    def _wrap(cls, batch: BitmapBatch) -> "RoaringBitmap":
        rb = cls.__new__(cls)
        rb._b = batch
        rb._snap = None
        return rb

    def _set(self, batch: BitmapBatch) -> None:
        """Replace the device state (mutation); host snapshots are dropped."""
        self._b = batch
        self._snap = None

    # --------------------------------------------------- host snapshots
    # The reference keeps `_keys` / `_containers` as Python lists
    # (bitmap.py:32-36).  Here the bitmap lives in HBM; these are host copies
    # taken on first access, for code that inspects them.  validate() checks
    # a snapshot against the device state, so a snapshot edited in place
    # reads as corruption (as the reference's validator would see it).
    def _snapshot(self):
        if self._snap is None:
            keys, conts = chunks_from_wire(self.serialize())
            self._snap = (keys, conts, list(keys))
        return self._snap

    @property
    def _keys(self) -> list:
        return self._snapshot()[0]

    @property
    def _containers(self) -> list:
        return self._snapshot()[1]

    # ------------------------------------------------------------- building
    @classmethod
    def from_values(cls, values) -> "RoaringBitmap":
        """Bulk-build from any iterable or array of 32-bit values (bitmap.py:40-62).
        The conversion mirrors the reference's: u64 via numpy, so a negative
        Python int raises OverflowError and anything above 2^32-1 ValueError."""
        arr = np.asarray(list(values) if not isinstance(values, np.ndarray) else values, dtype=np.uint64)
        return cls._wrap(BitmapBatch.from_values([arr]))

    @classmethod
    def deserialize(cls, data: bytes) -> "RoaringBitmap":
        return cls._wrap(BitmapBatch.from_wire([bytes(data)]))

    def serialize(self) -> bytes:
        return self._b.to_wire_list()[0]

    def copy(self) -> "RoaringBitmap":
        return RoaringBitmap._wrap(self._b.select([0]))

    # ------------------------------------------------------------ basic API
    def __len__(self) -> int:
        return int(self._b.cardinalities()[0])

    @property
    def cardinality(self) -> int:
        return len(self)

    def __bool__(self) -> bool:
        return int(self._b.container_counts()[0]) > 0

    def __eq__(self, other) -> bool:
        if not isinstance(other, RoaringBitmap):
            return NotImplemented
        return bool(self._b.equal(other._b, [0], [0])[0])

    def __repr__(self) -> str:
        return f"RoaringBitmap(card={len(self)}, chunks={int(self._b.container_counts()[0])})"

    def chunks(self) -> Iterator[tuple[int, Container]]:
        keys, conts = chunks_from_wire(self.serialize())
        return zip(keys, conts)

    def __contains__(self, v: int) -> bool:
        """Key lookup + container probe (bitmap.py:99-104) as one GPU query."""
        v = int(v)
        if not 0 <= v <= 0xFFFFFFFF:  # no such key in the reference either
            return False
        return bool(self._b.contains([v])[0])

    def contains_many(self, values) -> np.ndarray:
        """Batched membership: one GPU thread per query value."""
        return self._b.contains(values)

    # ------------------------------------------------------------- mutation
    def add(self, v: int) -> bool:
        """Insert v; True when the bitmap changed (bitmap.py:106-118).  The
        container re-typing of container_add (containers.py:271-319) is the
        OR result-type rule with a one-value array, so the update runs as a
        GPU pairwise OR against {v}."""
        v = int(v)
        if not 0 <= v <= 0xFFFFFFFF:
            raise ValueError("value out of 32-bit range")
        if v in self:
            return False
        self._set(self._b.pairwise("or", BitmapBatch.from_values([np.array([v], dtype=np.uint32)]), [0], [0]))
        return True

    def remove(self, v: int) -> bool:
        """Delete v; True when the bitmap changed (bitmap.py:120-134).  Runs as
        a GPU ANDNOT with {v}: container_remove's demotions (containers.py:322-
        367) and the dropping of an emptied chunk are that op's result rules."""
        v = int(v)
        if not 0 <= v <= 0xFFFFFFFF or v not in self:
            return False
        self._set(self._b.pairwise("andnot", BitmapBatch.from_values([np.array([v], dtype=np.uint32)]), [0], [0]))
        return True

    # ------------------------------------------------------------ iteration
    def to_array(self) -> np.ndarray:
        """All members, ascending, as uint32 (bitmap.py:136-144)."""
        return self._b.to_arrays()[0].copy()

    def __iter__(self) -> Iterator[int]:
        return iter(self.to_array().tolist())

    def for_each(self, visitor: Callable[[int], bool]) -> int:
        """Call visitor on members in ascending order while it returns True;
        returns the number visited (bitmap.py:152-166).  The values are
        extracted on the GPU; the visitor itself is host code."""
        count = 0
        for v in self.to_array().tolist():
            count += 1
            if not visitor(v):
                return count
        return count

    # ----------------------------------------------------------- set algebra
    def op(self, op: str, other: "RoaringBitmap") -> "RoaringBitmap":
        """and/or/andnot/xor between whole bitmaps; inputs untouched (bitmap.py:169-210)."""
        op_index(op)
        return RoaringBitmap._wrap(self._b.pairwise(op, other._b, [0], [0]))

    def op_cardinality(self, op: str, other: "RoaringBitmap") -> int:
        """Cardinality of op(self, other) without materializing it (bitmap.py:212-241)."""
        op_index(op)
        return int(self._b.pairwise_cardinality(op, other._b, [0], [0])[0])

    def __and__(self, other):
        return self.op("and", other)

    def __or__(self, other):
        return self.op("or", other)

    def __sub__(self, other):
        return self.op("andnot", other)

    def __xor__(self, other):
        return self.op("xor", other)

    # ---------------------------------------------------------- wide unions
    @staticmethod
    def union_many(bitmaps: Iterable["RoaringBitmap"]) -> "RoaringBitmap":
        """Sequential-fold semantics of bitmap.py:257-304, computed in one GPU pass."""
        bitmaps = list(bitmaps)
        if not bitmaps:
            return RoaringBitmap()
        batch = BitmapBatch.concat([b._b for b in bitmaps])
        return RoaringBitmap._wrap(batch.union_many())

    # ------------------------------------------------------- storage tuning
    def run_optimize(self) -> bool:
        """Re-pick each container's type with run candidacy (bitmap.py:308-316)."""
        self._snap = None
        return bool(self._b.run_optimize()[0])

    def shrink_to_fit(self) -> int:
        """Bytes reclaimed by trimming container capacity (bitmap.py:318-328),
        in the reference's accounting, where capacity == length here: 0.  The
        device side of the same idea happens too: an op result's pool, laid
        out by per-container upper bounds, is packed to its containers' bytes
        (rs_batch_info packs it)."""
        self._b.info()
        return 0

    def memory_bytes(self) -> tuple[int, int]:
        """(in-memory bytes, serialized bytes) under the reference's accounting
        (bitmap.py:330-353) with capacity == length (packed device pools)."""
        payload, _, types = self._b.stats()
        nc = sum(types.values())
        ser = 8 + 8 * nc + payload
        in_mem = 16 + 7 * nc + payload - 2 * types[3]  # run payload has no u16 count in memory
        return in_mem, ser

    # ------------------------------------------------------------ validation
    def validate(self) -> None:
        """Raise AssertionError if a structural invariant is broken: the image is
        re-ingested through the GPU decoder, which applies every serde check;
        a host snapshot (_keys / _containers) must still match the device."""
        try:
            BitmapBatch.from_wire([self.serialize()])
        except DecodeError as e:
            raise AssertionError(str(e)) from None
        if self._snap is not None:
            keys, conts, taken = self._snap
            assert all(0 <= k <= 0xFFFF for k in keys), "key outside 16 bits"
            assert all(a < b for a, b in zip(keys, keys[1:])), "keys not strictly increasing"
            assert keys == taken and len(conts) == len(keys), "key index differs from the bitmap"


__all__ = ["RoaringBitmap", "OPS"]
