"""Where does the e2e time go?  H2D bandwidth, ingest, ops, readback (C2)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth

buf, offs = synth.config2()
n = 1024
A_img = (buf[:int(offs[n])], offs[:n + 1].copy())
B_img = (buf[int(offs[n]):], (offs[n:] - offs[n]).astype(np.uint64))
pin = _lib.PinnedBuffer(A_img[0].nbytes)
pin.array[:] = A_img[0]
t = torch.from_numpy(pin.array)
dev = torch.empty(t.numel(), dtype=torch.uint8, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); dev.copy_(t, non_blocking=True); torch.cuda.synchronize()
    print(f"torch pinned H2D {t.numel()/1e9:.2f} GB: {(time.perf_counter()-t0)*1e3:.1f} ms -> {t.numel()/(time.perf_counter()-t0)/1e9:.1f} GB/s")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); h = dev.cpu(); torch.cuda.synchronize()
    print(f"torch D2H pageable: {t.numel()/(time.perf_counter()-t0)/1e9:.1f} GB/s")
for k in range(3):
    _lib.synchronize(); t0 = time.perf_counter()
    AA = rb.BitmapBatch.from_wire((pin.array, A_img[1]))
    _lib.synchronize(); t1 = time.perf_counter()
    print(f"from_wire(pinned, 2.15 GB): {(t1-t0)*1e3:.1f} ms")
BB = rb.BitmapBatch.from_wire(B_img)
for op in ("and", "or"):
    _lib.synchronize(); t0 = time.perf_counter()
    R = AA.pairwise(op, BB); c = R.cardinalities()
    _lib.synchronize(); t1 = time.perf_counter()
    s = R.wire_sizes().sum(); out = _lib.PinnedBuffer(int(s)); t2 = time.perf_counter()
    R.to_wire(out=out.array); t3 = time.perf_counter()
    print(f"{op}: op+cards {(t1-t0)*1e3:.1f} ms, to_wire {s/1e9:.2f} GB {(t3-t2)*1e3:.1f} ms")
