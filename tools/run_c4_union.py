"""One C4 union_many (for ncu captures of k_union_fold)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
buf, offs = synth.config4(nbitmaps=200)
Bt = rb.BitmapBatch.from_wire((buf, offs))
U = Bt.union_many()
_lib.synchronize()
print("ok", U.info())
