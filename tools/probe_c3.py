"""Per-class kernel times for config 3 (array x array container pairs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth

n = int(os.environ.get("C3_PAIRS", "1000000"))
buf, offs = synth.config3(npairs=n)
A = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, 0, n))
B = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, n, 2 * n))
import torch
dev_out = torch.empty(n, dtype=torch.int64, device="cuda")
names = ["array_pair_s", "array_pair_m", "array_pair_l", "array_pair_g", "generic_pair", "copy",
         "array_count_s", "array_count_m", "array_count_l"]
for op in ("and", "or", "andnot", "xor"):
    for kind in ("op", "count"):
        f = (lambda: A.container_pairwise(op, B)) if kind == "op" else (lambda: A.container_pairwise_cardinality_device(op, B, dev_out.data_ptr(), n))
        f(); _lib.synchronize()
        _lib.profile_reset(); _lib.profile(True)
        e0 = _lib.Event(); f(); e1 = _lib.Event(); _lib.synchronize()
        tot = e0.elapsed_ms(e1)
        parts = {k: _lib.profile_query(k) for k in names}
        _lib.profile(False)
        print(op, kind, f"total {tot:.3f} ms |", " ".join(f"{k}={v[0]:.3f}ms/{v[2]}" for k, v in parts.items() if v[1]))
