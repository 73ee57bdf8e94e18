"""Config-1 host path: kernel launches per API call and host microseconds per
launch, against the bare ctypes round trip (rs_batch_info)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import paper_1709_07821_b200 as rb
from paper_1709_07821_b200 import _lib
import workloads as synth
from paper_1709_07821_b200._lib import lib
buf, offs = synth.config1()
B = rb.BitmapBatch.from_wire((buf, offs))
n = 400
t0 = time.perf_counter()
for _ in range(n):
    B.info()
print(f"bare ctypes call (info): {1e6 * (time.perf_counter() - t0) / n:.1f} us")
for op in ("and", "or"):
    for _ in range(20):
        B.pairwise(op, B, [0], [1])
    _lib.synchronize()
    k0 = _lib.kernel_launches()
    t0 = time.perf_counter()
    for _ in range(n):
        B.pairwise(op, B, [0], [1])
    t1 = time.perf_counter()
    _lib.synchronize()
    print(f"{op}: {(_lib.kernel_launches() - k0) / n:.1f} launches/call, {1e6 * (t1 - t0) / n:.1f} us/call enqueue")
lib().rs_host_trace_dump()
