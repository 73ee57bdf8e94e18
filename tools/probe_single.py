"""Single-pair call costs (C1 shape): Python wrapper vs the bare C ABI call,
host read-back vs device output, per op."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
from paper_1709_07821_b200._lib import lib
import workloads as synth

buf, offs = synth.config1()
B = rb.BitmapBatch.from_wire((buf, offs))
L = lib()
ia = (C.c_uint32 * 1)(0)
ib = (C.c_uint32 * 1)(1)
out = np.zeros(1, dtype=np.uint64)
n = 2000


def rate(fn, sync=False):
    for _ in range(50):
        fn()
    _lib.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    _lib.synchronize()
    t2 = time.perf_counter()
    return 1e6 * (t1 - t0) / n, 1e6 * (t2 - t0) / n


for k, op in enumerate(("and", "or", "andnot", "xor")):
    print(op, "count: wrapper %.1f / %.1f us" % rate(lambda: B.pairwise_cardinality(op, B, [0], [1])),
          "| bare ABI %.1f / %.1f us" % rate(lambda: L.rs_pairwise_cardinality(k, B._h, B._h, ia, ib, 1,
                                                                            out.ctypes.data, 0)))
    h = C.c_void_p()
    print(op, "op: wrapper %.1f / %.1f us" % rate(lambda: B.pairwise(op, B, [0], [1])),
          "| bare ABI (leaks handles) %.1f / %.1f us" % rate(lambda: L.rs_pairwise(k, B._h, B._h, ia, ib, 1,
                                                                               C.byref(h))))
