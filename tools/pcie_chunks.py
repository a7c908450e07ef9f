"""Raw PCIe pipeline probe: r in (H2D) and z out (D2H) in chunks on two
streams, chunk c's D2H ordered after chunk c's H2D, no kernels.  Shows what
the copy engines can do for the host apply's shape (16.8 MB each way)."""
import sys
import time

import torch

n = 128 ** 3
r = torch.empty(n, dtype=torch.float64).pin_memory()
z = torch.empty(n, dtype=torch.float64).pin_memory()
rd = torch.empty(n, dtype=torch.float64, device="cuda")
zd = torch.empty(n, dtype=torch.float64, device="cuda")
sin, sout = torch.cuda.Stream(), torch.cuda.Stream()


def run(chunks_mb, lag=0):
    rows = [int(mb * (1 << 20) / 8) for mb in chunks_mb]
    b = [0]
    for x in rows:
        b.append(min(n, b[-1] + x))
    if b[-1] < n:
        b.append(n)
    evs = []
    with torch.cuda.stream(sin):
        for c in range(len(b) - 1):
            rd[b[c]:b[c + 1]].copy_(r[b[c]:b[c + 1]], non_blocking=True)
            e = torch.cuda.Event()
            e.record(sin)
            evs.append(e)
    with torch.cuda.stream(sout):
        for c in range(len(b) - 1):
            sout.wait_event(evs[min(len(evs) - 1, c + lag)])
            z[b[c]:b[c + 1]].copy_(zd[b[c]:b[c + 1]], non_blocking=True)
    torch.cuda.synchronize()


def t(fn, k=30):
    fn()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / k * 1e3


for sched in ([16.0], [2, 4, 4, 4, 2], [2, 3.67, 3.67, 3.66, 2, 1], [1] * 16, [0.5] * 32, [8, 8], [4] * 4):
    ms = t(lambda: run(sched))
    print(f"chunks {sched[:6]}{'...' if len(sched) > 6 else ''}: {ms:.4f} ms  ({2 * 8 * n / ms / 1e6:.1f} GB/s both ways, e2e-equiv {432677896 / ms / 1e6:.0f} GB/s)")
