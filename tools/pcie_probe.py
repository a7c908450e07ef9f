"""PCIe probe: pinned H2D / D2H bandwidth, alone and concurrently."""
import time
import torch

n = 2097152
h1 = torch.randn(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.randn(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
b = n * 8
h2d = t(lambda: d1.copy_(h1, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bo = t(both)
print(f"H2D {b/h2d/1e9:.1f} GB/s  D2H {b/d2h/1e9:.1f} GB/s  both-concurrent {2*b/bo/1e9:.1f} GB/s total ({bo*1e3:.3f} ms for 2x{b/1e6:.1f} MB)")
# chunked 16 x 1 MB
def chunked():
    for c in range(16):
        sl = slice(c * n // 16, (c + 1) * n // 16)
        d1[sl].copy_(h1[sl], non_blocking=True)
print(f"H2D chunked 16: {b/t(chunked)/1e9:.1f} GB/s")
