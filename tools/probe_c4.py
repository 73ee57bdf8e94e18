"""Per-class kernel times for config 4 (successive pairs of mixed bitmaps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth

buf, offs = synth.config4(nbitmaps=200)
Bt = rb.BitmapBatch.from_wire((buf, offs))
ia, ib = np.arange(199), np.arange(1, 200)
names = ["bitset_pair", "array_pair_s", "array_pair_m", "array_pair_l", "generic_pair", "probe_pair", "copy", "union_fold"]
for op in ("and", "or", "xor", "andnot"):
    Bt.pairwise(op, Bt, ia, ib); _lib.synchronize()
    _lib.profile_reset(); _lib.profile(True)
    e0 = _lib.Event(); R = Bt.pairwise(op, Bt, ia, ib); e1 = _lib.Event(); _lib.synchronize()
    tot = e0.elapsed_ms(e1)
    parts = {k: _lib.profile_query(k) for k in names}
    _lib.profile(False)
    print(op, f"total {tot:.3f} ms |", " ".join(f"{k}={v[0]:.3f}ms/{v[1]}" for k, v in parts.items() if v[1]),
          "| result", R.stats()[2])
_lib.profile_reset(); _lib.profile(True)
e0 = _lib.Event(); U = Bt.union_many(); e1 = _lib.Event(); _lib.synchronize()
print("union_many", f"total {e0.elapsed_ms(e1):.3f} ms", {k: _lib.profile_query(k) for k in ("union_fold",)})
