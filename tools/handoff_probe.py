"""Cross-stream hand-off latency: a chain of N (small H2D copy -> tiny
kernel) pairs on ONE stream vs the same chain alternating between a copy
stream and a compute stream through events (what the host pipelines do)."""
import time

import torch

N = 400
h = torch.ones(512, dtype=torch.float64).pin_memory()
d = torch.empty(512, dtype=torch.float64, device="cuda")
x = torch.zeros(1, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ev = [torch.cuda.Event() for _ in range(2 * N)]


def same():
    with torch.cuda.stream(s1):
        for _ in range(N):
            d.copy_(h, non_blocking=True)
            x.add_(1.0)


def cross():
    for i in range(N):
        with torch.cuda.stream(s1):
            if i:
                s1.wait_event(ev[2 * i - 1])
            d.copy_(h, non_blocking=True)
            ev[2 * i].record(s1)
        with torch.cuda.stream(s2):
            s2.wait_event(ev[2 * i])
            x.add_(1.0)
            ev[2 * i + 1].record(s2)


def kernels_cross():
    for i in range(N):
        with torch.cuda.stream(s1):
            if i:
                s1.wait_event(ev[2 * i - 1])
            x.add_(1.0)
            ev[2 * i].record(s1)
        with torch.cuda.stream(s2):
            s2.wait_event(ev[2 * i])
            x.add_(1.0)
            ev[2 * i + 1].record(s2)


def kernels_same():
    with torch.cuda.stream(s1):
        for _ in range(2 * N):
            x.add_(1.0)


for name, fn in (("copy+kernel same stream", same), ("copy+kernel cross streams", cross),
                 ("kernel+kernel same stream", kernels_same), ("kernel+kernel cross streams", kernels_cross)):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"{name}: {best / N * 1e6:.1f} us per pair", flush=True)
