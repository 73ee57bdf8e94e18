"""One C3 op of each kind (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
n = 1_000_000
buf, offs = synth.config3(npairs=n)
A = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, 0, n))
B = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, n, 2 * n))
for op in os.environ.get("RUN_OPS", "and,or,and,or").split(","):
    A.container_pairwise(op, B)
_lib.synchronize()
print("ok")
