import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2106_12836_b200 as S
A = S.laplacian_3d(128)
f = S.ilu_k(A, 0)
ML = S.sait_thr(S.DeviceCsr.upload(f.lower), S.lower_triangular, S.SaitThrParams(5e-2, 3))
MU = S.sait_thr(S.DeviceCsr.upload(f.upper), S.upper_triangular, S.SaitThrParams(5e-2, 3))
pair = S.SaitPairPreconditioner(ML, MU)
n = A.nrows
r = torch.from_numpy(S.uniform_pm1(1, n)).pin_memory(); z = torch.empty_like(r).pin_memory()
for _ in range(3): pair.apply(r.numpy(), z.numpy())
t0 = time.perf_counter()
for _ in range(20): pair.apply(r.numpy(), z.numpy())
print("ms per host apply", (time.perf_counter() - t0) / 20 * 1e3)
