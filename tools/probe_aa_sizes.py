"""Array x array container ops at fixed pair sizes: per-value cost of the
large-pair kernels vs per-pair overhead (tools only)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import torch


def images(rng, npairs, n):
    hdr = b"ROAR" + (1).to_bytes(4, "little")
    out = []
    for _ in range(npairs):
        v = np.sort(rng.choice(65536, n, replace=False)).astype("<u2")
        out.append(hdr + (0).to_bytes(2, "little") + bytes([1, 0]) + n.to_bytes(4, "little") + v.tobytes())
    return out


rng = np.random.default_rng(1)
SIZES = ((300, 200000), (1000, 60000), (4096, 15000))
if len(sys.argv) > 1:
    SIZES = [SIZES[int(a)] for a in sys.argv[1].split(",")]
for n, npairs in SIZES:
    A = rb.BitmapBatch.from_wire(images(rng, npairs, n))
    B = rb.BitmapBatch.from_wire(images(rng, npairs, n))
    dev = torch.empty(npairs, dtype=torch.int64, device="cuda")
    res = {}
    for op in ("and", "or"):
        for kind in ("op", "count"):
            fn = (lambda: A.container_pairwise(op, B)) if kind == "op" else \
                (lambda: A.container_pairwise_cardinality_device(op, B, dev.data_ptr(), npairs))
            for _ in range(3):
                fn()
            _lib.synchronize()
            e0 = _lib.Event()
            for _ in range(5):
                fn()
            e1 = _lib.Event()
            ms = e0.elapsed_ms(e1) / 5
            res[f"{op}_{kind}"] = ms
    vals = 2 * n * npairs
    print(f"n={n} pairs={npairs}: " + ", ".join(f"{k} {v:.3f} ms ({v * 1e6 / vals:.3f} ns/value, "
                                                  f"{v * 1e6 / npairs:.0f} ns/pair)" for k, v in res.items()), flush=True)
