"""C5 all-pairs call: per-phase host wall times (RS_TRACE=1 synchronizes per
phase) on the last of several calls, plus the live kernel times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
buf, offs = synth.config5()
B = rb.BitmapBatch.from_wire((buf, offs))
for _ in range(3):
    B.all_pairs_cardinality()
_lib.synchronize()
_lib.profile_reset(); _lib.profile(True)
t0 = time.perf_counter()
B.all_pairs_cardinality()
_lib.synchronize()
print(f"wall {1e3 * (time.perf_counter() - t0):.3f} ms")
for k in ("densify", "allpairs_umma", "allpairs"):
    print(k, _lib.profile_query(k))
