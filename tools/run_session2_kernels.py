"""One call each of the paths reworked in round 2's second session (for one
ncu capture): a C1 single-pair op and count (one launch each), a C4 AND
(A-indexed join, per-pair compaction), a C3 AND (dynamic large-pair kernel,
staged galloping pairs) and a C5 all-pairs call (densify)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
buf, offs = synth.config1()
B1 = rb.BitmapBatch.from_wire((buf, offs))
B1.pairwise("and", B1, [0], [1])
B1.pairwise_cardinality("or", B1, [0], [1])
buf, offs = synth.config4(nbitmaps=200)
B4 = rb.BitmapBatch.from_wire((buf, offs))
B4.pairwise("and", B4, np.arange(199), np.arange(1, 200))
n = 1_000_000
buf, offs = synth.config3(npairs=n)
A3 = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, 0, n))
B3 = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, n, 2 * n))
A3.container_pairwise("and", B3)
buf, offs = synth.config5()
B5 = rb.BitmapBatch.from_wire((buf, offs))
B5.all_pairs_cardinality()
_lib.synchronize()
print("ok")
