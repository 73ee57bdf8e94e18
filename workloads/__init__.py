"""Seeded synthetic workloads for the five BASELINE.json configs (bench/test inputs).

Workload generation only -- not part of the set-operation path.  The C
generator (synth.c, OpenMP) emits reference wire images, built as the
reference harness builds its structures (from_values, plus run_optimize where
the config calls for it).  Seeds default to 1..5, one per config.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "libworkloads.so")
_lib = None


def build() -> str:
    src = os.path.join(_HERE, "synth.c")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return LIB


def use_library(path: str) -> None:
    """Load the generator from another library that links synth.c (the
    bench's reference arm uses oracle/liboracle.so, so that arm maps no
    other library of this repository)."""
    global _lib, LIB
    LIB = path
    _lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB if os.path.exists(LIB) else build())
        P, I64, U64, D, I = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int
        pp = C.POINTER(C.c_void_p)
        L.syn_uniform.argtypes = [U64, I64, U64, U64, pp, pp]
        L.syn_bernoulli.argtypes = [U64, I64, I, D, D, pp, pp, P]
        L.syn_zipf_pairs.argtypes = [U64, I64, D, pp, pp]
        L.syn_mixed.argtypes = [U64, I64, I, D, D, D, D, D, pp, pp]
        L.syn_clusters.argtypes = [U64, I64, U64, I, U64, U64, D, pp, pp]
        L.syn_free.argtypes = [P]
        L.syn_num_threads.restype = I
        _lib = L
    return _lib


def _take(buf: C.c_void_p, offs: C.c_void_p, n: int):
    L = lib()
    o = np.ctypeslib.as_array(C.cast(offs, C.POINTER(C.c_uint64)), shape=(n + 1,)).copy()
    total = int(o[-1])
    b = np.empty(max(total, 1), dtype=np.uint8)
    if total:
        C.memmove(b.ctypes.data, buf, total)
    L.syn_free(buf)
    L.syn_free(offs)
    return b[:total], o


def config1(seed: int = 1, count: int = 100_000, universe: int = 1 << 22, nbitmaps: int = 2):
    """C1: bitmaps of `count` distinct uniform values in [0, universe)."""
    b, o = C.c_void_p(), C.c_void_p()
    if lib().syn_uniform(seed, nbitmaps, count, universe, C.byref(b), C.byref(o)):
        raise MemoryError("synth config1")
    return _take(b, o, nbitmaps)


def config2(seed: int = 2, npairs: int = 1024, nchunks: int = 256, plo: float = 0.1, phi: float = 0.5):
    """C2: 2*npairs Bernoulli(p) bitmaps, p ~ U[plo, phi] per bitmap; pair p = (p, npairs+p)."""
    b, o = C.c_void_p(), C.c_void_p()
    if lib().syn_bernoulli(seed, 2 * npairs, nchunks, plo, phi, C.byref(b), C.byref(o), None):
        raise MemoryError("synth config2")
    return _take(b, o, 2 * npairs)


def config3(seed: int = 3, npairs: int = 1_000_000, s: float = 1.2):
    """C3: one-container array pairs, Zipf(s) sizes; images [0,n) are A, [n,2n) are B."""
    b, o = C.c_void_p(), C.c_void_p()
    if lib().syn_zipf_pairs(seed, npairs, s, C.byref(b), C.byref(o)):
        raise MemoryError("synth config3")
    return _take(b, o, 2 * npairs)


def config4(seed: int = 4, nbitmaps: int = 200, nkeys: int = 2000, dlo: float = 2.0 ** -12, dhi: float = 0.9,
            run_frac: float = 0.3, gap_mean: float = 256.0, len_mean: float = 64.0):
    """C4: mixed-container collection (run-optimized)."""
    b, o = C.c_void_p(), C.c_void_p()
    if lib().syn_mixed(seed, nbitmaps, nkeys, dlo, dhi, run_frac, gap_mean, len_mean, C.byref(b), C.byref(o)):
        raise MemoryError("synth config4")
    return _take(b, o, nbitmaps)


def config5(seed: int = 5, nbitmaps: int = 512, universe: int = 1 << 26, nclusters: int = 8,
            smin: int = 1 << 14, smax: int = 1 << 17, sigma: float = float(1 << 18)):
    """C5: clustered bitmaps for all-pairs Jaccard (run-optimized)."""
    b, o = C.c_void_p(), C.c_void_p()
    if lib().syn_clusters(seed, nbitmaps, universe, nclusters, smin, smax, sigma, C.byref(b), C.byref(o)):
        raise MemoryError("synth config5")
    return _take(b, o, nbitmaps)


def slice_images(buf: np.ndarray, offs: np.ndarray, lo: int, hi: int) -> tuple[np.ndarray, np.ndarray]:
    """Images [lo, hi) of a (buf, offs) image set, as a new (buf, offs) view."""
    a, b = int(offs[lo]), int(offs[hi])
    return buf[a:b], (offs[lo:hi + 1] - offs[lo]).astype(np.uint64)
