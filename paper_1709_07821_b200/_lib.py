"""ctypes binding of the C ABI in include/roaring_b200.h (libroaring_b200.so).

The library is built in-tree by __graft_entry__.build() (nvcc, sm_100a).  There
is no fallback: if the shared object is missing, or no CUDA device is present,
every compute call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libroaring_b200.so")

RS_OK, RS_EOP, RS_EDECODE, RS_EVALUE, RS_EARG, RS_ECUDA, RS_ENOMEM, RS_ESHAPE = range(8)


class DecodeError(ValueError):
    """Malformed wire image; carries the byte offset (serde.py:55-60)."""

    def __init__(self, offset: int, message: str):
        super().__init__(f"at byte {offset}: {message}")
        self.offset = offset


class RoaringCudaError(RuntimeError):
    """CUDA failure or no device: the product path never falls back to the CPU."""


_lib = None
_lock = threading.Lock()


def _declare(L):
    P, U64, I64, I32 = C.c_void_p, C.c_uint64, C.c_int64, C.c_int
    pp = C.POINTER(C.c_void_p)
    sig = {
        "rs_last_error": ([], C.c_char_p),
        "rs_last_error_offset": ([], I64),
        "rs_last_error_index": ([], I64),
        "rs_version": ([], C.c_char_p),
        "rs_set_device": ([I32], I32),
        "rs_set_stream": ([P], I32),
        "rs_get_stream": ([], P),
        "rs_synchronize": ([], I32),
        "rs_host_alloc": ([pp, U64], I32),
        "rs_host_free": ([P], I32),
        "rs_event_record": ([pp], I32),
        "rs_event_elapsed": ([P, P, C.POINTER(C.c_float)], I32),
        "rs_event_destroy": ([P], I32),
        "rs_kernel_launches": ([], U64),
        "rs_batch_from_wire": ([P, P, U64, pp], I32),
        "rs_batch_from_wire_async": ([P, P, U64, pp], I32),
        "rs_batch_from_wire_device": ([P, P, U64, pp], I32),
        "rs_batch_wait": ([P], I32),
        "rs_batch_from_u32": ([P, P, U64, I32, pp], I32),
        "rs_batch_free": ([P], I32),
        "rs_batch_info": ([P, P, P, P], I32),
        "rs_batch_len": ([P], U64),
        "rs_batch_cardinalities": ([P, P], I32),
        "rs_batch_cardinalities_device": ([P, P], I32),
        "rs_batch_container_counts": ([P, P], I32),
        "rs_batch_concat": ([P, U64, pp], I32),
        "rs_batch_select": ([P, P, U64, pp], I32),
        "rs_batch_key_range": ([P, C.c_uint32, C.c_uint32, pp], I32),
        "rs_batch_key_histogram": ([P, P], I32),
        "rs_batch_wire_sizes": ([P, P], I32),
        "rs_batch_to_wire": ([P, P, U64, P], I32),
        "rs_batch_to_wire_async": ([P, P, U64, P, pp], I32),
        "rs_event_synchronize": ([P], I32),
        "rs_event_query": ([P], I32),
        "rs_batch_to_u32": ([P, P, U64, P], I32),
        "rs_batch_equal": ([P, P, P, P, U64, P], I32),
        "rs_batch_digests": ([P, P, I32], I32),
        "rs_batch_contains": ([P, P, P, U64, P], I32),
        "rs_pairwise": ([I32, P, P, P, P, U64, pp], I32),
        "rs_pairwise_cardinality": ([I32, P, P, P, P, U64, P, I32], I32),
        "rs_container_pairwise": ([I32, P, P, P, P, U64, pp], I32),
        "rs_container_pairwise_cardinality": ([I32, P, P, P, P, U64, P, I32], I32),
        "rs_union_many": ([P, P, U64, pp], I32),
        "rs_all_pairs_cardinality": ([P, P, P], I32),
        "rs_batch_run_optimize": ([P, P], I32),
        "rs_batch_stats": ([P, P, P, P], I32),
        "rs_profile_enable": ([I32], I32),
        "rs_profile_reset": ([], I32),
        "rs_profile_query": ([C.c_char_p, P, P, P], I32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


def lib():
    """Load libroaring_b200.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: build the CUDA library first "
                        "(python -c 'import __graft_entry__ as g; g.build()')")
                _lib = _declare(C.CDLL(LIB_PATH))
    return _lib


def check(rc: int) -> None:
    """Map a C ABI status to the reference's exception types."""
    if rc == RS_OK:
        return
    L = lib()
    msg = L.rs_last_error().decode(errors="replace")
    if rc == RS_EDECODE:
        off = int(L.rs_last_error_offset())
        prefix = f"at byte {off}: "
        raise DecodeError(off, msg[len(prefix):] if msg.startswith(prefix) else msg)
    if rc in (RS_EOP, RS_EVALUE, RS_EARG, RS_ESHAPE):
        raise ValueError(msg)
    if rc == RS_ENOMEM:
        raise MemoryError(msg)
    raise RoaringCudaError(msg)


def kernel_launches() -> int:
    return int(lib().rs_kernel_launches())


def set_device(device: int) -> None:
    check(lib().rs_set_device(int(device)))


def set_stream(stream_handle: int | None) -> None:
    check(lib().rs_set_stream(C.c_void_p(stream_handle or 0)))


def synchronize() -> None:
    check(lib().rs_synchronize())


def profile(on: bool) -> None:
    """Bracket the hot kernels with CUDA events on the launch stream."""
    check(lib().rs_profile_enable(1 if on else 0))


def profile_reset() -> None:
    check(lib().rs_profile_reset())


def profile_query(name: str):
    """(total ms, launches, work items) of the kernel tagged `name`."""
    ms, n, it = C.c_double(), C.c_uint64(), C.c_uint64()
    check(lib().rs_profile_query(name.encode(), C.byref(ms), C.byref(n), C.byref(it)))
    return float(ms.value), int(n.value), int(it.value)


class Event:
    """CUDA event recorded on the library stream."""

    def __init__(self):
        self._e = C.c_void_p()
        check(lib().rs_event_record(C.byref(self._e)))

    def elapsed_ms(self, later: "Event") -> float:
        ms = C.c_float()
        check(lib().rs_event_elapsed(self._e, later._e, C.byref(ms)))
        return float(ms.value)

    def __del__(self):
        try:
            if self._e:
                lib().rs_event_destroy(self._e)
        except Exception:
            pass


class Completion:
    """A CUDA event handed out by an asynchronous call (rs_batch_to_wire_async):
    wait() blocks until the work behind it has finished; done() polls."""

    def __init__(self, handle: C.c_void_p):
        self._e = handle

    def wait(self) -> None:
        check(lib().rs_event_synchronize(self._e))

    def done(self) -> bool:
        rc = lib().rs_event_query(self._e)
        if rc == 1:
            return False
        check(rc)
        return True

    def __del__(self):
        try:
            if self._e:
                lib().rs_event_destroy(self._e)
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host memory (cudaMallocHost) exposed as a numpy array."""

    def __init__(self, nbytes: int):
        import numpy as np
        self._p = C.c_void_p()
        check(lib().rs_host_alloc(C.byref(self._p), max(int(nbytes), 16)))
        self.nbytes = int(nbytes)
        self.array = np.ctypeslib.as_array(C.cast(self._p, C.POINTER(C.c_uint8)), shape=(max(self.nbytes, 16),))[
            :self.nbytes]

    def __del__(self):
        try:
            if self._p:
                lib().rs_host_free(self._p)
        except Exception:
            pass


class _PinnedView:
    """Owner of one pooled page-locked block, exported to numpy through the
    array interface.  Every array made from it -- slices, views, `arr[:m]` --
    reaches this object through its `.base` chain, so the block goes back to
    the pool only when the last of them dies."""

    __slots__ = ("__array_interface__", "_buf", "__weakref__")

    def __init__(self, buf: "PinnedBuffer", nbytes: int):
        self._buf = buf
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                    "data": (buf._p.value, False), "version": 3}


class _PinnedPool:
    """Recycled page-locked result arrays for large device->host readbacks.

    A fresh numpy array is pageable: the copy goes through the driver's staging
    buffers (~11 GB/s measured) and first-touch page faults.  Arrays from
    `empty()` view a cached cudaMallocHost block (power-of-two size class);
    when the last view of an array dies its block goes back to the pool, so a
    repeated call reads back at PCIe speed into already-resident pages.  The
    caller owns the returned array like any numpy array: the block's lifetime
    is tied to a `_PinnedView` owner that every derived view references."""

    MIN_BYTES = 1 << 16          # smaller results: plain numpy (pinning buys nothing)
    MAX_CACHED = 256 << 20       # free bytes kept for reuse

    def __init__(self):
        self._free: dict[int, list] = {}
        self._cached = 0
        self._mu = threading.Lock()

    def empty(self, n: int, dtype):
        import numpy as np
        import weakref
        dt = np.dtype(dtype)
        nbytes = max(int(n), 1) * dt.itemsize
        if nbytes < self.MIN_BYTES:
            return np.empty(max(int(n), 1), dtype=dt)
        size = 1 << (nbytes - 1).bit_length()
        with self._mu:
            lst = self._free.get(size)
            buf = lst.pop() if lst else None
            if buf is not None:
                self._cached -= size
        if buf is None:
            buf = PinnedBuffer(size)
        owner = _PinnedView(buf, nbytes)
        weakref.finalize(owner, self._release, size, buf)
        return np.asarray(owner).view(dt)

    def _release(self, size: int, buf) -> None:
        with self._mu:
            if self._cached + size <= self.MAX_CACHED:
                self._free.setdefault(size, []).append(buf)
                self._cached += size
                return
        del buf  # over the cap: cudaFreeHost via PinnedBuffer.__del__


pinned_pool = _PinnedPool()
