"""One C3 AND count (container_pairwise_cardinality) for ncu captures of k_aa_large_count."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
n = 1_000_000
op = sys.argv[1] if len(sys.argv) > 1 else "and"
buf, offs = synth.config3(npairs=n)
A = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, 0, n))
B = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, n, 2 * n))
c = A.container_pairwise_cardinality(op, B)
R = A.container_pairwise(op, B)
_lib.synchronize()
print("ok", int(c.sum()))
