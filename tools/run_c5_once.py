"""One C5 all-pairs run (for ncu captures of the tensor-core tiles)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
buf, offs = synth.config5()
B = rb.BitmapBatch.from_wire((buf, offs))
inter, uni = B.all_pairs_cardinality()
_lib.synchronize()
print("ok", int(inter.sum()))
