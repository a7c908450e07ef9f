"""Pair apply throughput: 100 applies issued from Python vs the same 100
applies replayed from a captured CUDA graph (is the step host-bound?)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_12836_b200 as S  # noqa: E402

A = S.laplacian_3d(128)
f = S.ilu_k(A, 0)
P = S.SaitPairPreconditioner(S.sait_thr(S.DeviceCsr.upload(f.lower), S.lower_triangular, S.SaitThrParams(5e-2, 3)),
                             S.sait_thr(S.DeviceCsr.upload(f.upper), S.upper_triangular, S.SaitThrParams(5e-2, 3)))
n = A.nrows
R = torch.rand((100, n), dtype=torch.float64, device="cuda")
Z = torch.empty_like(R)
s = torch.cuda.Stream()


def step():
    for i in range(100):
        P.apply(R[i], Z[i])


with torch.cuda.stream(s):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        step()
    b.record()
    torch.cuda.synchronize()
    print("python-issued: us per pair", a.elapsed_time(b) / 1000 * 1000)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    print("graph replay: us per pair", a.elapsed_time(b) / 1000 * 1000)
