"""Copy-engine gaps between back-to-back pinned H2D copies on one stream:
one large copy vs k copies of size/k, with and without an event recorded
between them (what the block pipeline does)."""
import time

import torch

n = 100 * 2097152
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
evs = [torch.cuda.Event() for _ in range(400)]


def run(k, ev):
    m = n // k
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for i in range(k):
            d[i * m:(i + 1) * m].copy_(h[i * m:(i + 1) * m], non_blocking=True)
            if ev:
                evs[i % 400].record(s)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for k in (1, 10, 50, 100, 200, 400):
    for ev in (False, True):
        run(k, ev)
        t = min(run(k, ev) for _ in range(3))
        print(f"k={k:4d} event={int(ev)}: {n * 8 / t / 1e9:6.1f} GB/s  per-copy {t / k * 1e6:8.1f} us", flush=True)
