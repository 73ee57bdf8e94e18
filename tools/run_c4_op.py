"""One C4 op over the 199 successive pairs (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
op = sys.argv[1] if len(sys.argv) > 1 else "and"
buf, offs = synth.config4(nbitmaps=200)
Bt = rb.BitmapBatch.from_wire((buf, offs))
R = Bt.pairwise(op, Bt, np.arange(199), np.arange(1, 200))
_lib.synchronize()
print("ok", R.stats()[2])
