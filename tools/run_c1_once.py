"""C1 step (4 ops + 4 counts on one pair) for launch-list captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
buf, offs = synth.config1()
B = rb.BitmapBatch.from_wire((buf, offs))
for rep in range(3):
    for op in ("and", "or", "andnot", "xor"):
        B.pairwise(op, B, [0], [1])
    for op in ("and", "or", "andnot", "xor"):
        B.pairwise_cardinality(op, B, [0], [1])
_lib.synchronize()
print("ok")
