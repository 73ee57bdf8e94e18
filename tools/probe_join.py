"""AND / ANDNOT batches of successive config-4-style bitmaps at several
(pairs, keys per bitmap) shapes: median CUDA-event time per call (A/B of the
per-pair join against the A-indexed join: RS_PER_PAIR=-1 | 0)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
out = {}
for nb, nk in ((9, 16), (33, 64), (65, 64), (129, 32), (257, 32), (16385, 4), (4097, 16), (1025, 64), (297, 256), (65, 1024)):
    buf, offs = synth.config4(seed=7, nbitmaps=nb, nkeys=nk)
    B = rb.BitmapBatch.from_wire((buf, offs))
    ia, ib = np.arange(nb - 1), np.arange(1, nb)
    for op in ("and", "andnot"):
        for _ in range(3):
            B.pairwise(op, B, ia, ib)
        _lib.synchronize()
        ts = []
        for _ in range(9):
            e0 = _lib.Event(); B.pairwise(op, B, ia, ib); e1 = _lib.Event()
            ts.append(e0.elapsed_ms(e1))
        out[f"{nb - 1}x{nk} {op}"] = round(statistics.median(ts), 4)
print(out)
