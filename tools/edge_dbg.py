import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1709_07821_b200 as pkg
from paper_1709_07821_b200 import _lib
RB = pkg.RoaringBitmap
empty = RB()
full = RB.from_values(np.arange(0, 1 << 17, dtype=np.uint32)); full.run_optimize()
one = RB.from_values([65535])
cases = {"empty": empty, "full": full, "one": one, "four": RB.from_values([0, 65535, 65536, (1 << 32) - 1])}
for na, a in cases.items():
    for nb, b in cases.items():
        for op in ("and", "or", "andnot", "xor"):
            try:
                r = a.op(op, b); _lib.synchronize(); r.serialize()
                c = a.op_cardinality(op, b)
            except Exception as e:
                print("FAIL", na, nb, op, str(e)[:100]); sys.exit(1)
print("all ok")
