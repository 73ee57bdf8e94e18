"""Kernel split of union_many (C4) and all-pairs cardinality (C5)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth

buf, offs = synth.config4()
B4 = rb.BitmapBatch.from_wire((buf, offs))
buf, offs = synth.config5()
B5 = rb.BitmapBatch.from_wire((buf, offs))
for name, f, parts in (("union_many C4", lambda: B4.union_many(), ["union_fold"]),
                       ("all_pairs C5", lambda: B5.all_pairs_cardinality(), ["densify", "allpairs", "allpairs_umma"])):
    f(); _lib.synchronize()
    for rep in range(2):
        _lib.profile_reset(); _lib.profile(True)
        e0 = _lib.Event(); f(); e1 = _lib.Event(); _lib.synchronize()
        q = {k: _lib.profile_query(k) for k in parts}
        _lib.profile(False)
        print(name, f"total {e0.elapsed_ms(e1):.3f} ms |", " ".join(f"{k}={v[0]:.3f}ms x{v[1]}" for k, v in q.items()))
