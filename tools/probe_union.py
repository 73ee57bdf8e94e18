"""C4 union_many: median CUDA-event time over repetitions (tuning A/B; set
RS_UNION_SPLIT etc. in the environment), and a digest parity check."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
from paper_1709_07821_b200.batch import fold_digests
import workloads as synth
import json
buf, offs = synth.config4(nbitmaps=200)
Bt = rb.BitmapBatch.from_wire((buf, offs))
want = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "tests/golden/config_digests.json")))["C4"]["union_many"]
U = Bt.union_many()
got = fold_digests(U.digests())
del U
ts = []
for _ in range(3):
    Bt.union_many()
_lib.synchronize()
for _ in range(15):
    e0 = _lib.Event(); Bt.union_many(); e1 = _lib.Event()
    ts.append(e0.elapsed_ms(e1))
print(f"split={os.environ.get('RS_UNION_SPLIT', '-')} union_many median {statistics.median(ts):.3f} ms "
      f"min {min(ts):.3f} parity {'ok' if format(got, '016x') == want or got == want else ('MISMATCH', got, want)}")
