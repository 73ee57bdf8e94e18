"""One materialized C2 op (default AND) for a targeted ncu capture of k_bb_op."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth

op = sys.argv[1] if len(sys.argv) > 1 else "and"
npairs = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
buf, offs = synth.config2(npairs=npairs)
A = rb.BitmapBatch.from_wire((buf[:int(offs[npairs])], offs[:npairs + 1].copy()))
B = rb.BitmapBatch.from_wire((buf[int(offs[npairs]):], (offs[npairs:] - offs[npairs]).astype(np.uint64)))
R = A.pairwise(op, B)
_lib.synchronize()
print(op, "ok", R.stats()[2])
