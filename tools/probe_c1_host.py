"""Host-side cost of one C1 call: enqueue rate (no sync) vs synchronous round trip."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
buf, offs = synth.config1()
B = rb.BitmapBatch.from_wire((buf, offs))
import torch
dev = torch.empty(1, dtype=torch.int64, device="cuda")
for op in ("and", "or"):
    for _ in range(20):
        B.pairwise(op, B, [0], [1])
    _lib.synchronize()
    n = 500
    t0 = time.perf_counter()
    for _ in range(n):
        R = B.pairwise(op, B, [0], [1])
    t1 = time.perf_counter()
    _lib.synchronize()
    t2 = time.perf_counter()
    print(f"{op}: enqueue {1e6*(t1-t0)/n:.1f} us/call, drained at {1e6*(t2-t0)/n:.1f} us/call")
    t0 = time.perf_counter()
    for _ in range(n):
        B.pairwise_cardinality_device(op, B, dev.data_ptr(), 1, [0], [1])
    t1 = time.perf_counter(); _lib.synchronize(); t2 = time.perf_counter()
    print(f"{op} count (device out): enqueue {1e6*(t1-t0)/n:.1f} us/call, drained {1e6*(t2-t0)/n:.1f} us/call")
    t0 = time.perf_counter()
    for _ in range(n):
        B.pairwise_cardinality(op, B, [0], [1])
    t1 = time.perf_counter()
    print(f"{op} count (host out, sync): {1e6*(t1-t0)/n:.1f} us/call")
# Python-side fixed costs
L = _lib.lib()
t0 = time.perf_counter()
for _ in range(5000):
    L.rs_batch_len(B._h)
print(f"bare ctypes call: {1e6*(time.perf_counter()-t0)/5000:.2f} us")
from paper_1709_07821_b200.batch import _u32_or_none
t0 = time.perf_counter()
for _ in range(5000):
    _u32_or_none([0]); _u32_or_none([1])
print(f"two index conversions: {1e6*(time.perf_counter()-t0)/5000:.2f} us")
