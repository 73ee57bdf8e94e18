"""C4 per-op host enqueue time vs drained time (is the op host- or GPU-bound?)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
buf, offs = synth.config4(nbitmaps=200)
Bt = rb.BitmapBatch.from_wire((buf, offs))
ia, ib = np.arange(199), np.arange(1, 200)
for op in ("and", "or", "andnot", "xor"):
    for _ in range(5):
        Bt.pairwise(op, Bt, ia, ib)
    _lib.synchronize()
    n = 30
    k0 = _lib.kernel_launches()
    t0 = time.perf_counter()
    rs = []
    for _ in range(n):
        e0 = _lib.Event(); R = Bt.pairwise(op, Bt, ia, ib); e1 = _lib.Event()
        rs.append((e0, e1)); del R
    t1 = time.perf_counter()
    _lib.synchronize()
    t2 = time.perf_counter()
    ev = sorted(a.elapsed_ms(b) for a, b in rs)
    print(f"{op}: {(_lib.kernel_launches() - k0) / n:.1f} launches, enqueue {1e3 * (t1 - t0) / n:.3f} ms/call, "
          f"drained {1e3 * (t2 - t0) / n:.3f} ms/call, event median {ev[n // 2]:.3f} ms")
