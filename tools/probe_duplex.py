"""PCIe duplex probe: pinned H2D alone, D2H alone, and both at once on two streams."""
import time
import torch

n = 2 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if h2d:
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for _ in range(2):
    a, b, c = run(True, False), run(False, True), run(True, True)
print(f"H2D {n / a / 1e9:.1f} GB/s  D2H {n / b / 1e9:.1f} GB/s  both: {c * 1e3:.1f} ms "
      f"(serial would be {(a + b) * 1e3:.1f} ms, overlap {2 * n / c / 1e9:.1f} GB/s total)")
