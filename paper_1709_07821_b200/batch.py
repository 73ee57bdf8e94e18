"""BitmapBatch: a device-resident collection of Roaring bitmaps (the batched API).

One BitmapBatch owns one ``rs_batch`` of the C ABI (include/roaring_b200.h):
a CSR container table plus a 16-byte aligned payload pool in HBM.  Every
method is one batched call into hand-written sm_100a kernels; the reference's
per-pair semantics (bitmap.py / containers.py under
/root/reference/pkg/src/roaringset) hold for every pair of the batch.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib
from .containers import op_index


def _u32_or_none(idx, n_expected=None):
    """Pair indices as a u32 buffer for the C ABI: (owner, address).  Short
    Python sequences (the one-pair calls of the RoaringBitmap API) skip numpy:
    its array construction and min/max cost ~3.5 us per call, as much as a
    kernel launch."""
    if idx is None:
        return None, None
    if isinstance(idx, (list, tuple)) and len(idx) <= 16:
        for v in idx:
            if not 0 <= v <= 0xFFFFFFFF:
                raise ValueError("bitmap index out of range")
        buf = (C.c_uint32 * max(len(idx), 1))(*idx)
        return buf, C.addressof(buf)
    a = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    if a.size and (a.min() < 0 or a.max() > 0xFFFFFFFF):
        raise ValueError("bitmap index out of range")
    a = a.astype(np.uint32)
    return a, a.ctypes.data


def _images(images):
    """list[bytes] | (uint8 buf, uint64 offs) -> (buf, offs) numpy arrays."""
    if isinstance(images, tuple) and len(images) == 2 and isinstance(images[0], np.ndarray):
        buf, offs = images
        return np.ascontiguousarray(buf, dtype=np.uint8), np.ascontiguousarray(offs, dtype=np.uint64)
    images = list(images)
    offs = np.zeros(len(images) + 1, dtype=np.uint64)
    if images:
        np.cumsum([len(x) for x in images], out=offs[1:])
    buf = np.frombuffer(b"".join(images), dtype=np.uint8) if images else np.zeros(1, np.uint8)
    return buf, offs


_FOLD_K = np.uint64(0x9E3779B97F4A7C15)


def fold_digests(values) -> int:
    """One 64-bit digest of an ordered sequence of u64 (per-bitmap content
    digests, or counts): sum_i mix(v_i + (i+1) * K) mod 2^64, mix the
    SplitMix64 finalizer -- order-sensitive, so a permuted batch differs."""
    z = np.ascontiguousarray(values, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        z += np.arange(1, len(z) + 1, dtype=np.uint64) * _FOLD_K
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
        return int(z.sum(dtype=np.uint64))


class BitmapBatch:
    __slots__ = ("_h", "_keep", "__weakref__")

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        self._keep = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().rs_batch_free(h)
            except Exception:
                pass
            self._h = None

    # ------------------------------------------------------------ building
    @classmethod
    def from_wire(cls, images, *, deferred: bool = False) -> "BitmapBatch":
        """serde.deserialize (serde.py:87-169) of many images at once.

        deferred=True returns as soon as the transfer is queued: the payload
        bytes move on the library's copy stream (overlapping kernels already
        queued) and their checks are read back by wait() -- or by the first
        call that returns values to the host.  The image buffer must stay
        alive and untouched until then; pinned memory (PinnedBuffer) makes the
        copy asynchronous."""
        buf, offs = _images(images)
        h = C.c_void_p()
        fn = lib().rs_batch_from_wire_async if deferred else lib().rs_batch_from_wire
        check(fn(buf.ctypes.data, offs.ctypes.data, len(offs) - 1, C.byref(h)))
        b = cls(h)
        if deferred:
            b._keep = buf  # the copy engine reads it after we return
        return b

    @classmethod
    def from_wire_device(cls, buf_ptr: int, offs_ptr: int, n: int) -> "BitmapBatch":
        """serde.deserialize of n wire images already in device memory: buf_ptr /
        offs_ptr are device pointers (uint8 bytes; uint64[n+1] offsets, relative
        to the byte at buf_ptr for offs[0]) -- e.g. a torch CUDA tensor's
        data_ptr().  The descriptor walk runs on the device too."""
        h = C.c_void_p()
        check(lib().rs_batch_from_wire_device(C.c_void_p(buf_ptr), C.c_void_p(offs_ptr), int(n), C.byref(h)))
        return cls(h)

    def wait(self) -> "BitmapBatch":
        """Raise DecodeError if the deferred payload checks failed."""
        check(lib().rs_batch_wait(self._h))
        return self

    @classmethod
    def from_values(cls, arrays) -> "BitmapBatch":
        """RoaringBitmap.from_values (bitmap.py:40-62) for each array."""
        parts = []
        for a in arrays:
            a = np.asarray(a)
            if a.size:
                a = np.asarray(a, dtype=np.uint64)
                if int(a.max()) > 0xFFFFFFFF:
                    raise ValueError("values must fit in 32 bits")
            parts.append(a.astype(np.uint32, copy=False).ravel())
        offs = np.zeros(len(parts) + 1, dtype=np.uint64)
        if parts:
            np.cumsum([p.size for p in parts], out=offs[1:])
        vals = np.concatenate(parts) if parts else np.zeros(0, np.uint32)
        return cls.from_values_flat(vals, offs)

    @classmethod
    def from_values_flat(cls, values: np.ndarray, offs: np.ndarray) -> "BitmapBatch":
        v = np.ascontiguousarray(values, dtype=np.uint32)
        o = np.ascontiguousarray(offs, dtype=np.uint64)
        h = C.c_void_p()
        check(lib().rs_batch_from_u32(v.ctypes.data if v.size else None, o.ctypes.data, len(o) - 1, 0, C.byref(h)))
        return cls(h)

    @staticmethod
    def concat(batches) -> "BitmapBatch":
        batches = list(batches)
        arr = (C.c_void_p * max(len(batches), 1))(*[b._h for b in batches])
        h = C.c_void_p()
        check(lib().rs_batch_concat(arr, len(batches), C.byref(h)))
        return BitmapBatch(h)

    def select(self, idx) -> "BitmapBatch":
        """Deep copy of bitmaps idx (RoaringBitmap.copy, bitmap.py:71-73)."""
        a = np.ascontiguousarray(np.asarray(idx, dtype=np.uint64))
        h = C.c_void_p()
        check(lib().rs_batch_select(self._h, a.ctypes.data, a.size, C.byref(h)))
        return BitmapBatch(h)

    def key_range(self, lo: int, hi: int) -> "BitmapBatch":
        """Every bitmap restricted to chunk keys [lo, hi) (multi-GPU key-range
        sharding; dist.py)."""
        h = C.c_void_p()
        check(lib().rs_batch_key_range(self._h, int(lo), int(hi), C.byref(h)))
        return BitmapBatch(h)

    def key_histogram(self) -> np.ndarray:
        """Containers per chunk key over the batch (u64[65536])."""
        out = np.zeros(65536, dtype=np.uint64)
        check(lib().rs_batch_key_histogram(self._h, out.ctypes.data))
        return out

    # ------------------------------------------------------------- queries
    def info(self):
        nb, nc, pb = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().rs_batch_info(self._h, C.byref(nb), C.byref(nc), C.byref(pb)))
        return int(nb.value), int(nc.value), int(pb.value)

    def __len__(self) -> int:
        return int(lib().rs_batch_len(self._h))

    def stats(self):
        """(payload bytes, descriptor bytes, {tag: count}) in the SURVEY 8(d) accounting."""
        pb, db = C.c_uint64(), C.c_uint64()
        tc = np.zeros(4, dtype=np.uint64)
        check(lib().rs_batch_stats(self._h, C.byref(pb), C.byref(db), tc.ctypes.data))
        return int(pb.value), int(db.value), {1: int(tc[1]), 2: int(tc[2]), 3: int(tc[3])}

    def cardinalities(self) -> np.ndarray:
        out = np.zeros(max(len(self), 1), dtype=np.uint64)
        check(lib().rs_batch_cardinalities(self._h, out.ctypes.data))
        return out[:len(self)]

    def cardinalities_device(self, dst_ptr: int) -> None:
        """Per-bitmap cardinalities into device memory at dst_ptr (u64[n]),
        stream-ordered, without synchronizing."""
        check(lib().rs_batch_cardinalities_device(self._h, dst_ptr))

    def container_counts(self) -> np.ndarray:
        out = np.zeros(max(len(self), 1), dtype=np.uint64)
        check(lib().rs_batch_container_counts(self._h, out.ctypes.data))
        return out[:len(self)]

    # -------------------------------------------------------------- export
    def wire_sizes(self) -> np.ndarray:
        out = np.zeros(max(len(self), 1), dtype=np.uint64)
        check(lib().rs_batch_wire_sizes(self._h, out.ctypes.data))
        return out[:len(self)]

    def to_wire(self, out: np.ndarray | None = None):
        """serde.serialize of every bitmap -> (uint8 buffer, uint64 offsets)."""
        n = len(self)
        total = int(self.wire_sizes().sum())
        buf = out if out is not None else np.empty(max(total, 1), dtype=np.uint8)
        offs = np.zeros(n + 1, dtype=np.uint64)
        check(lib().rs_batch_to_wire(self._h, buf.ctypes.data, buf.nbytes, offs.ctypes.data))
        return buf[:total], offs

    def to_wire_async(self, out: np.ndarray):
        """serde.serialize of every bitmap into `out` (uint8, ideally
        page-locked: PinnedBuffer) without waiting for the transfer.
        Returns (offsets, completion): offsets are final on return, the bytes
        are in `out` once completion.wait() returns.  `out` must stay alive
        until then; this batch may be freed at once."""
        n = len(self)
        offs = _lib.pinned_pool.empty(n + 1, np.uint64)
        e = C.c_void_p()
        check(lib().rs_batch_to_wire_async(self._h, out.ctypes.data, out.nbytes, offs.ctypes.data, C.byref(e)))
        return offs, _lib.Completion(e)

    def to_wire_list(self) -> list[bytes]:
        buf, offs = self.to_wire()
        return [buf[int(offs[i]):int(offs[i + 1])].tobytes() for i in range(len(offs) - 1)]

    def to_arrays_flat(self):
        """RoaringBitmap.to_array of every bitmap -> (uint32 values, uint64 offsets)."""
        n = len(self)
        total = int(self.cardinalities().sum())
        vals = np.empty(max(total, 1), dtype=np.uint32)
        offs = np.zeros(n + 1, dtype=np.uint64)
        check(lib().rs_batch_to_u32(self._h, vals.ctypes.data, vals.size, offs.ctypes.data))
        return vals[:total], offs

    def to_arrays(self) -> list[np.ndarray]:
        vals, offs = self.to_arrays_flat()
        return [vals[int(offs[i]):int(offs[i + 1])] for i in range(len(offs) - 1)]

    def digests(self) -> np.ndarray:
        """64-bit content digest per bitmap, computed on the device (equal
        bitmaps, equal digests; rs_batch_digests)."""
        out = np.zeros(max(len(self), 1), dtype=np.uint64)
        check(lib().rs_batch_digests(self._h, out.ctypes.data, 0))
        return out[:len(self)]

    def digest(self) -> int:
        """fold_digests of the per-bitmap content digests: one u64 for the
        whole batch's exact content."""
        return fold_digests(self.digests())

    def equal(self, other: "BitmapBatch", ia=None, ib=None) -> np.ndarray:
        """Type-sensitive equality per pair (bitmap.py:87-91)."""
        n = self._npairs(other, ia, ib)
        a, pa = _u32_or_none(ia)
        b, pb = _u32_or_none(ib)
        out = np.zeros(max(n, 1), dtype=np.uint8)
        check(lib().rs_batch_equal(self._h, other._h, pa, pb, n, out.ctypes.data))
        return out[:n].astype(bool)

    def contains(self, values, bitmaps=None) -> np.ndarray:
        """hit[q] = values[q] in bitmap bitmaps[q] (all bitmap 0 when None);
        RoaringBitmap.__contains__ (bitmap.py:99-104), one GPU thread per query."""
        v = np.ascontiguousarray(np.asarray(values, dtype=np.int64).reshape(-1))
        if v.size and (v.min() < 0 or v.max() > 0xFFFFFFFF):
            raise ValueError("values must fit in 32 bits")
        v = v.astype(np.uint32)
        n = len(v)
        b, pb = _u32_or_none(bitmaps)
        if b is not None and len(b) != n:
            raise ValueError("bitmaps and values differ in length")
        out = np.zeros(max(n, 1), dtype=np.uint8)
        check(lib().rs_batch_contains(self._h, pb, v.ctypes.data, n, out.ctypes.data))
        return out[:n].astype(bool)

    # ------------------------------------------------------------ hot path
    def _npairs(self, other, ia, ib, n=None):
        """Pair count of a call, checked against the index arrays the C ABI
        reads (npairs u32 each): ia and ib must have equal lengths, and an
        explicit n must not exceed either of them."""
        la = None if ia is None else len(ia)
        lb = None if ib is None else len(ib)
        if la is not None and lb is not None and la != lb:
            raise ValueError(f"ia and ib differ in length ({la} != {lb})")
        if n is None:
            return la if la is not None else lb if lb is not None else min(len(self), len(other))
        n = int(n)
        if n < 0 or (la is not None and n > la) or (lb is not None and n > lb):
            raise ValueError(f"n={n} exceeds the pair index arrays")
        return n

    def pairwise(self, op: str, other: "BitmapBatch", ia=None, ib=None) -> "BitmapBatch":
        """Bitmap p of the result = self[ia[p]] op other[ib[p]] (bitmap.py:169-210)."""
        k = op_index(op)
        n = self._npairs(other, ia, ib)
        a, pa = _u32_or_none(ia)
        b, pb = _u32_or_none(ib)
        h = C.c_void_p()
        check(lib().rs_pairwise(k, self._h, other._h, pa, pb, n, C.byref(h)))
        return BitmapBatch(h)

    def pairwise_cardinality(self, op: str, other: "BitmapBatch", ia=None, ib=None) -> np.ndarray:
        """|self[ia[p]] op other[ib[p]]| (bitmap.py:212-241)."""
        k = op_index(op)
        n = self._npairs(other, ia, ib)
        a, pa = _u32_or_none(ia)
        b, pb = _u32_or_none(ib)
        out = np.zeros(max(n, 1), dtype=np.uint64)
        check(lib().rs_pairwise_cardinality(k, self._h, other._h, pa, pb, n, out.ctypes.data, 0))
        return out[:n]

    def pairwise_cardinality_device(self, op: str, other: "BitmapBatch", dev_out_ptr: int, n: int,
                                    ia=None, ib=None) -> None:
        """Asynchronous variant writing u64 counts to a device pointer."""
        k = op_index(op)
        n = self._npairs(other, ia, ib, n)
        a, pa = _u32_or_none(ia)
        b, pb = _u32_or_none(ib)
        check(lib().rs_pairwise_cardinality(k, self._h, other._h, pa, pb, n, C.c_void_p(dev_out_ptr), 1))

    def container_pairwise(self, op: str, other: "BitmapBatch", ia=None, ib=None) -> "BitmapBatch":
        """containers.py:450-529 over one-container bitmaps, batched."""
        k = op_index(op)
        n = self._npairs(other, ia, ib)
        a, pa = _u32_or_none(ia)
        b, pb = _u32_or_none(ib)
        h = C.c_void_p()
        check(lib().rs_container_pairwise(k, self._h, other._h, pa, pb, n, C.byref(h)))
        return BitmapBatch(h)

    def container_pairwise_cardinality_device(self, op: str, other: "BitmapBatch", dev_out_ptr: int, n: int,
                                              ia=None, ib=None) -> None:
        """Asynchronous variant writing u64 counts to a device pointer."""
        k = op_index(op)
        n = self._npairs(other, ia, ib, n)
        a, pa = _u32_or_none(ia)
        b, pb = _u32_or_none(ib)
        check(lib().rs_container_pairwise_cardinality(k, self._h, other._h, pa, pb, n, C.c_void_p(dev_out_ptr), 1))

    def container_pairwise_cardinality(self, op: str, other: "BitmapBatch", ia=None, ib=None) -> np.ndarray:
        """containers.py:554-570, batched."""
        k = op_index(op)
        n = self._npairs(other, ia, ib)
        a, pa = _u32_or_none(ia)
        b, pb = _u32_or_none(ib)
        out = np.zeros(max(n, 1), dtype=np.uint64)
        check(lib().rs_container_pairwise_cardinality(k, self._h, other._h, pa, pb, n, out.ctypes.data, 0))
        return out[:n]

    def union_many(self, idx=None) -> "BitmapBatch":
        """RoaringBitmap.union_many (bitmap.py:257-304) over bitmaps idx (default: all, in order)."""
        n = len(idx) if idx is not None else len(self)
        a = np.ascontiguousarray(np.asarray(idx, dtype=np.uint64)) if idx is not None else None
        h = C.c_void_p()
        check(lib().rs_union_many(self._h, a.ctypes.data if a is not None else None, n, C.byref(h)))
        return BitmapBatch(h)

    def all_pairs_cardinality(self):
        """(|B_i ∩ B_j|, |B_i ∪ B_j|) for all i<j in row-major order."""
        n = len(self)
        m = n * (n - 1) // 2
        # every entry is written by the call; large results land in recycled
        # page-locked memory (PCIe-rate readback, no first-touch faults)
        inter = _lib.pinned_pool.empty(max(m, 1), np.uint64)
        uni = _lib.pinned_pool.empty(max(m, 1), np.uint64)
        check(lib().rs_all_pairs_cardinality(self._h, inter.ctypes.data, uni.ctypes.data))
        return inter[:m], uni[:m]

    def run_optimize(self) -> np.ndarray:
        """RoaringBitmap.run_optimize (bitmap.py:308-316) on every bitmap, in place."""
        n = len(self)
        out = np.zeros(max(n, 1), dtype=np.uint8)
        check(lib().rs_batch_run_optimize(self._h, out.ctypes.data))
        return out[:n].astype(bool)

    def bitmap(self, i: int):
        from .bitmap import RoaringBitmap
        return RoaringBitmap._wrap(self.select([i]))

    def __repr__(self) -> str:
        nb, nc, pb = self.info()
        return f"BitmapBatch(bitmaps={nb}, containers={nc}, pool_bytes={pb})"


_ = _lib  # re-exported module for callers wanting stream/event helpers
