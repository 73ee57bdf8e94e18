"""C2 per-call medians (CUDA events, REPS reps): the 4 materialized ops and 4
counts over the 1,024 bitset pairs (tuning A/B; parity is in the tests and in
bench.py's digests)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
import torch
npairs = 1024
REPS = int(os.environ.get("REPS", "9"))
buf, offs = synth.config2(npairs=npairs)
A = rb.BitmapBatch.from_wire((buf[:int(offs[npairs])], offs[:npairs + 1].copy()))
B = rb.BitmapBatch.from_wire((buf[int(offs[npairs]):], (offs[npairs:] - offs[npairs]).astype(np.uint64)))
dev = torch.empty(npairs, dtype=torch.int64, device="cuda")
out = {}
for op in ("and", "or", "andnot", "xor"):
    for kind in ("op", "count"):
        f = (lambda: A.pairwise(op, B)) if kind == "op" else \
            (lambda: A.pairwise_cardinality_device(op, B, dev.data_ptr(), npairs))
        for _ in range(2):
            f()
        _lib.synchronize()
        ts = []
        for _ in range(REPS):
            e0 = _lib.Event(); f(); e1 = _lib.Event()
            ts.append(e0.elapsed_ms(e1))
        out[op + ("" if kind == "op" else "_c")] = round(statistics.median(ts), 3)
print(out, "sum", round(sum(out.values()), 3))
