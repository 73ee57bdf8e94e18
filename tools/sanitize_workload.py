"""Small end-to-end workload touching every kernel family, for compute-sanitizer
(tools/sanitize.sh): golden bitmap pairs (all container mixes, all ops,
counts), container pairs incl. empty images, union_many, all-pairs counts on
the tensor-core tiles and the CUDA-core tiles, from_values (sorted and not),
run_optimize, exports (sync, async, u32, digests), membership, key ranges,
deferred ingest with a malformed image.  Inputs are small so racecheck and
synccheck finish in minutes."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1709_07821_b200 as rb  # noqa: E402
from paper_1709_07821_b200 import _lib  # noqa: E402
from tests.golden_io import load  # noqa: E402
import workloads as synth  # noqa: E402

OPS = ("and", "or", "andnot", "xor")
g = load()
n = 24
A = rb.BitmapBatch.from_wire([g.wire(a) for a in g["pair_a"][:n]])
B = rb.BitmapBatch.from_wire([g.wire(b) for b in g["pair_b"][:n]])
for op in OPS:
    R = A.pairwise(op, B)
    R.to_wire_list()
    R.digests()
    R.info()
    A.pairwise_cardinality(op, B)
CA = rb.BitmapBatch.from_wire([g.wire(a) for a in g["cont_a"][:n]] + [b"ROAR\x00\x00\x00\x00"])
CB = rb.BitmapBatch.from_wire([b"ROAR\x00\x00\x00\x00"] + [g.wire(b) for b in g["cont_b"][:n]])
for op in OPS:
    CA.container_pairwise(op, CB).to_wire_list()
    CA.container_pairwise_cardinality(op, CB)
buf, offs = synth.config4(seed=3, nbitmaps=6, nkeys=48)
C4 = rb.BitmapBatch.from_wire((buf, offs))
C4.union_many().to_wire_list()
C4.pairwise("or", C4, [0, 1, 2], [3, 4, 5]).to_wire_list()
C4.key_range(1000, 40000).to_wire_list()
os.environ["RS_ALLPAIRS_UMMA_MIN"] = "2"
C4.all_pairs_cardinality()
del os.environ["RS_ALLPAIRS_UMMA_MIN"]
C4.all_pairs_cardinality()
rng = np.random.default_rng(1)
V = rb.BitmapBatch.from_values([rng.integers(0, 1 << 20, 5000), np.arange(70000, dtype=np.uint32)])
V.run_optimize()
V.to_arrays()
V.contains([5, 70001, 1 << 30])
pin = _lib.PinnedBuffer(1 << 24)
offs2, done = A.pairwise("xor", B).to_wire_async(pin.array)
done.wait()
bad = bytearray(g.wire(g["pair_a"][0]))
D = rb.BitmapBatch.from_wire((np.frombuffer(bytes(bad), np.uint8), np.array([0, len(bad)], np.uint64)), deferred=True)
D.pairwise("and", A, [0], [0])
D.wait()
_lib.synchronize()
print("sanitize workload ok")
