"""One C2 bench step (4 pairwise + 4 pairwise_cardinality_device) after a
warm-up step, for launch-list captures (ncu --metrics gpu__time_duration.sum)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth

OPS = ("and", "or", "andnot", "xor")
n = 1024
buf, offs = synth.config2(npairs=n)
A = rb.BitmapBatch.from_wire((buf[:int(offs[n])], offs[:n + 1].copy()))
B = rb.BitmapBatch.from_wire((buf[int(offs[n]):], (offs[n:] - offs[n]).astype(np.uint64)))
counts = torch.empty(n, dtype=torch.int64, device="cuda")
for rep in range(2):
    for op in OPS:
        R = A.pairwise(op, B)
        del R
    for op in OPS:
        A.pairwise_cardinality_device(op, B, counts.data_ptr(), n)
_lib.synchronize()
print("ok")
