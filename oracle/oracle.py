"""ctypes wrapper over the C restatement of the reference (roaring_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as the
checker) and bench.py's cpu_baseline / ``--impl reference`` legs.  The product
package never imports this module.

All data crosses as reference wire images (serde.py:3-10 in
/root/reference/pkg/src/roaringset), so a parity check is a byte comparison
that covers values and container types at once.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
OPS = ("and", "or", "andnot", "xor")  # kernels/_shared.py:8


class OracleDecodeError(ValueError):
    """Mirror of serde.DecodeError (serde.py:55-60)."""

    def __init__(self, offset: int, message: str):
        super().__init__(f"at byte {offset}: {message}")
        self.offset = offset
        self.message = message


def build() -> str:
    src = os.path.join(_HERE, "roaring_oracle.c")
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P, S, I64, U64 = C.c_void_p, C.c_size_t, C.c_int64, C.c_uint64
        pp = C.POINTER(C.c_void_p)
        L.orc_last_error.restype = C.c_char_p
        L.orc_last_error_offset.restype = I64
        L.orc_free.argtypes = [P]
        L.orc_check.argtypes = [P, S]
        L.orc_roundtrip.argtypes = [P, S, pp, C.POINTER(S)]
        L.orc_op.argtypes = [C.c_int, P, S, P, S, pp, C.POINTER(S)]
        L.orc_op_cardinality.argtypes = [C.c_int, P, S, P, S, C.POINTER(I64)]
        L.orc_container_pairwise_cardinality.argtypes = [C.c_int, P, S, P, S, C.POINTER(I64)]
        L.orc_union_many.argtypes = [P, P, C.c_int32, pp, C.POINTER(S)]
        L.orc_from_values.argtypes = [P, I64, pp, C.POINTER(S)]
        L.orc_run_optimize.argtypes = [P, S, pp, C.POINTER(S), C.POINTER(C.c_int)]
        L.orc_to_array.argtypes = [P, S, pp, C.POINTER(I64)]
        L.orc_cardinality.argtypes = [P, S]
        L.orc_cardinality.restype = I64
        L.orc_op_batch.argtypes = [C.c_int, P, P, P, P, P, P, I64, P, P, C.c_int]
        L.orc_op_cardinality_batch.argtypes = [C.c_int, P, P, P, P, P, P, I64, P, C.c_int]
        L.orc_container_card_batch.argtypes = [C.c_int, P, P, P, P, P, P, I64, P, C.c_int]
        L.orc_all_pairs_and.argtypes = [P, P, I64, P, P, I64, P, C.c_int]
        L.orc_num_threads.restype = C.c_int
        L.orc_batch_load.argtypes = [P, P, I64, C.c_int]
        L.orc_batch_load.restype = P
        L.orc_batch_free.argtypes = [P]
        L.orc_batch_run.argtypes = [C.c_int, C.c_int, P, P, P, P, I64, P, C.c_int]
        L.orc_digest_images.argtypes = [P, P, I64, P, C.c_int]
        L.orc_batch_digest.argtypes = [C.c_int, C.c_int, P, P, P, P, I64, P, C.c_int]
        L.orc_union_digest.argtypes = [P, P]
        _lib = L
    return _lib


def num_threads() -> int:
    return int(lib().orc_num_threads())


def _op_index(op: str) -> int:
    if op not in OPS:
        raise ValueError(f"unknown op {op!r}")
    return OPS.index(op)


def _raise(rc: int):
    L = lib()
    msg = L.orc_last_error().decode()
    if rc == -1:
        raise OracleDecodeError(int(L.orc_last_error_offset()), msg)
    raise ValueError(msg)


def _take_bytes(ptr: C.c_void_p, n: int) -> bytes:
    out = C.string_at(ptr, n)
    lib().orc_free(ptr)
    return out


def check(wire: bytes) -> None:
    """Validate a wire image exactly as serde.deserialize does (serde.py:87-169)."""
    rc = lib().orc_check(wire, len(wire))
    if rc:
        _raise(rc)


def roundtrip(wire: bytes) -> bytes:
    p, n = C.c_void_p(), C.c_size_t()
    rc = lib().orc_roundtrip(wire, len(wire), C.byref(p), C.byref(n))
    if rc:
        _raise(rc)
    return _take_bytes(p, n.value)


def op(op_name: str, wa: bytes, wb: bytes) -> bytes:
    """serialize(deserialize(wa).op(op_name, deserialize(wb))) -- bitmap.py:169-210."""
    p, n = C.c_void_p(), C.c_size_t()
    rc = lib().orc_op(_op_index(op_name), wa, len(wa), wb, len(wb), C.byref(p), C.byref(n))
    if rc:
        _raise(rc)
    return _take_bytes(p, n.value)


def op_cardinality(op_name: str, wa: bytes, wb: bytes) -> int:
    """bitmap.py:212-241."""
    c = C.c_int64()
    rc = lib().orc_op_cardinality(_op_index(op_name), wa, len(wa), wb, len(wb), C.byref(c))
    if rc:
        _raise(rc)
    return int(c.value)


def container_pairwise_cardinality(op_name: str, wa: bytes, wb: bytes) -> int:
    """containers.py:554-570 over two one-container images."""
    c = C.c_int64()
    rc = lib().orc_container_pairwise_cardinality(_op_index(op_name), wa, len(wa), wb, len(wb),
                                                  C.byref(c))
    if rc:
        _raise(rc)
    return int(c.value)


def concat(wires) -> tuple[np.ndarray, np.ndarray]:
    """Concatenate wire images -> (uint8 buffer, uint64 offsets[n+1])."""
    lens = np.fromiter((len(w) for w in wires), dtype=np.uint64, count=len(wires))
    offs = np.zeros(len(wires) + 1, dtype=np.uint64)
    np.cumsum(lens, out=offs[1:])
    buf = np.frombuffer(b"".join(wires), dtype=np.uint8) if wires else np.zeros(1, np.uint8)
    return buf, offs


def union_many(wires) -> bytes:
    """bitmap.py:257-304."""
    buf, offs = concat(list(wires))
    p, n = C.c_void_p(), C.c_size_t()
    rc = lib().orc_union_many(buf.ctypes.data, offs.ctypes.data, len(offs) - 1, C.byref(p),
                              C.byref(n))
    if rc:
        _raise(rc)
    return _take_bytes(p, n.value)


def from_values(values) -> bytes:
    """bitmap.py:40-62 (values in any order, duplicates allowed)."""
    v = np.ascontiguousarray(np.asarray(values, dtype=np.uint64))
    p, n = C.c_void_p(), C.c_size_t()
    rc = lib().orc_from_values(v.ctypes.data, v.size, C.byref(p), C.byref(n))
    if rc:
        _raise(rc)
    return _take_bytes(p, n.value)


def run_optimize(wire: bytes) -> tuple[bytes, bool]:
    """bitmap.py:308-316."""
    p, n, ch = C.c_void_p(), C.c_size_t(), C.c_int()
    rc = lib().orc_run_optimize(wire, len(wire), C.byref(p), C.byref(n), C.byref(ch))
    if rc:
        _raise(rc)
    return _take_bytes(p, n.value), bool(ch.value)


def to_array(wire: bytes) -> np.ndarray:
    """bitmap.py:136-144."""
    p, n = C.c_void_p(), C.c_int64()
    rc = lib().orc_to_array(wire, len(wire), C.byref(p), C.byref(n))
    if rc:
        _raise(rc)
    out = np.frombuffer(C.string_at(p, 4 * n.value), dtype=np.uint32).copy()
    lib().orc_free(p)
    return out


def cardinality(wire: bytes) -> int:
    return int(lib().orc_cardinality(wire, len(wire)))


def _i64(x, n=None):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.int64))
    if n is not None:
        assert a.size == n
    return a


def op_batch(op_name, bufA, offA, bufB, offB, ia, ib, threads: int = 0) -> list[bytes]:
    """Materialized op for each pair p: A[ia[p]] op B[ib[p]] -> list of wire images."""
    ia, ib = _i64(ia), _i64(ib)
    n = ia.size
    outs = (C.c_void_p * max(n, 1))()
    lens = np.zeros(max(n, 1), dtype=np.uint64)
    rc = lib().orc_op_batch(_op_index(op_name), bufA.ctypes.data, offA.ctypes.data,
                            bufB.ctypes.data, offB.ctypes.data, ia.ctypes.data, ib.ctypes.data,
                            n, outs, lens.ctypes.data, threads)
    if rc:
        raise RuntimeError("oracle op_batch failed to decode an input")
    return [_take_bytes(outs[p], int(lens[p])) for p in range(n)]


def op_cardinality_batch(op_name, bufA, offA, bufB, offB, ia, ib, threads: int = 0) -> np.ndarray:
    ia, ib = _i64(ia), _i64(ib)
    out = np.zeros(ia.size, dtype=np.int64)
    rc = lib().orc_op_cardinality_batch(_op_index(op_name), bufA.ctypes.data, offA.ctypes.data,
                                        bufB.ctypes.data, offB.ctypes.data, ia.ctypes.data,
                                        ib.ctypes.data, ia.size, out.ctypes.data, threads)
    if rc:
        raise RuntimeError("oracle op_cardinality_batch failed to decode an input")
    return out


def container_card_batch(op_name, bufA, offA, bufB, offB, ia, ib, threads: int = 0) -> np.ndarray:
    ia, ib = _i64(ia), _i64(ib)
    out = np.zeros(ia.size, dtype=np.int64)
    rc = lib().orc_container_card_batch(_op_index(op_name), bufA.ctypes.data, offA.ctypes.data,
                                        bufB.ctypes.data, offB.ctypes.data, ia.ctypes.data,
                                        ib.ctypes.data, ia.size, out.ctypes.data, threads)
    if rc:
        raise RuntimeError("oracle container_card_batch failed")
    return out


def all_pairs_and(buf, offs, pi, pj, threads: int = 0) -> np.ndarray:
    pi, pj = _i64(pi), _i64(pj)
    out = np.zeros(pi.size, dtype=np.int64)
    rc = lib().orc_all_pairs_and(buf.ctypes.data, offs.ctypes.data, len(offs) - 1,
                                 pi.ctypes.data, pj.ctypes.data, pi.size, out.ctypes.data, threads)
    if rc:
        raise RuntimeError("oracle all_pairs_and failed")
    return out


class Session:
    """Bitmaps deserialized once into the oracle's in-memory form; run() times
    only the restated reference algorithm (the harness protocol,
    bench/harness.py:205-239)."""

    KINDS = {"op": 0, "op_cardinality": 1, "container_pairwise": 2,
             "container_pairwise_cardinality": 3}

    def __init__(self, buf, offs, threads: int = 0):
        buf = np.ascontiguousarray(buf, dtype=np.uint8)
        offs = np.ascontiguousarray(offs, dtype=np.uint64)
        self._h = lib().orc_batch_load(buf.ctypes.data, offs.ctypes.data, len(offs) - 1, threads)
        if not self._h:
            raise RuntimeError("oracle session: an image failed to decode")

    def run(self, op_name: str, kind: str, other: "Session", ia, ib, threads: int = 0) -> np.ndarray:
        ia, ib = _i64(ia), _i64(ib)
        out = np.zeros(max(ia.size, 1), dtype=np.int64)
        lib().orc_batch_run(_op_index(op_name), self.KINDS[kind], self._h, other._h, ia.ctypes.data,
                            ib.ctypes.data, ia.size, out.ctypes.data, threads)
        return out[:ia.size]

    def digests(self, op_name: str, kind: str, other: "Session", ia, ib, threads: int = 0) -> np.ndarray:
        """Content digests (roaring_oracle.c "content digests") of the results
        of op / container_pairwise over the pairs, without serializing them."""
        ia, ib = _i64(ia), _i64(ib)
        out = np.zeros(max(ia.size, 1), dtype=np.uint64)
        lib().orc_batch_digest(_op_index(op_name), self.KINDS[kind], self._h, other._h, ia.ctypes.data,
                               ib.ctypes.data, ia.size, out.ctypes.data, threads)
        return out[:ia.size]

    def union_digest(self) -> int:
        out = np.zeros(1, dtype=np.uint64)
        lib().orc_union_digest(self._h, out.ctypes.data)
        return int(out[0])

    def __del__(self):
        try:
            lib().orc_batch_free(self._h)
        except Exception:
            pass


def digest_images(buf, offs, threads: int = 0) -> np.ndarray:
    """Content digest of each wire image (roaring_oracle.c "content digests")."""
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    offs = np.ascontiguousarray(offs, dtype=np.uint64)
    n = len(offs) - 1
    out = np.zeros(max(n, 1), dtype=np.uint64)
    rc = lib().orc_digest_images(buf.ctypes.data, offs.ctypes.data, n, out.ctypes.data, threads)
    if rc:
        _raise(-1)
    return out[:n]
