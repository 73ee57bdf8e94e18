"""C3 per-call medians (CUDA events, 7 reps): 4 container_pairwise + 4
container_pairwise_cardinality_device over the 1 M pairs (tuning A/B; the
parity of these calls is in tests/test_gpu_fullscale.py)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
import torch
n = 1_000_000
REPS = int(os.environ.get("REPS", "7"))
SPREAD = os.environ.get("SPREAD") == "1"
buf, offs = synth.config3(npairs=n)
A = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, 0, n))
B = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, n, 2 * n))
dev = torch.empty(n, dtype=torch.int64, device="cuda")
out = {}
for op in ("and", "or", "andnot", "xor"):
    for kind in ("op", "count"):
        f = (lambda: A.container_pairwise(op, B)) if kind == "op" else \
            (lambda: A.container_pairwise_cardinality_device(op, B, dev.data_ptr(), n))
        for _ in range(2):
            f()
        _lib.synchronize()
        ts = []
        for _ in range(REPS):
            e0 = _lib.Event(); f(); e1 = _lib.Event()
            ts.append(e0.elapsed_ms(e1))
        out[op + ("" if kind == "op" else "_c")] = round(statistics.median(ts), 3)
        if SPREAD:
            print(op, kind, " ".join(f"{x:.3f}" for x in ts))
print(out, "sum", round(sum(out.values()), 3))
