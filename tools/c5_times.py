"""C5 all-pairs call: median CUDA-event time of REPS calls, and a digest check
of both count arrays against the cached oracle digests (tuning A/B)."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
from paper_1709_07821_b200.batch import fold_digests
import workloads as synth
REPS = int(os.environ.get("REPS", "9"))
buf, offs = synth.config5()
B = rb.BitmapBatch.from_wire((buf, offs))
inter, uni = B.all_pairs_cardinality()
want = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "tests/golden/config_digests.json")))["C5"]
got = {"inter": format(fold_digests(np.asarray(inter, dtype=np.uint64)), "016x"),
       "union": format(fold_digests(np.asarray(uni, dtype=np.uint64)), "016x")}
ok = all(got[k] == want.get(k) for k in got)
for _ in range(2):
    B.all_pairs_cardinality()
_lib.synchronize()
ts = []
for _ in range(REPS):
    e0 = _lib.Event(); B.all_pairs_cardinality(); e1 = _lib.Event()
    ts.append(e0.elapsed_ms(e1))
print(f"corner={os.environ.get('RS_ALLPAIRS_CORNER', '0')} C5 median {statistics.median(ts):.3f} ms "
      f"min {min(ts):.3f} parity {'ok' if ok else ('MISMATCH', got, want)}")
