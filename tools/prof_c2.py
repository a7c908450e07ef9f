"""Short C2 driver for ncu: build both factors on device, then `--applies`
pair applies on device vectors.  Not a benchmark (no timing printed)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_12836_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=128)
ap.add_argument("--applies", type=int, default=5)
ap.add_argument("--block", type=int, default=0, help="also run block applies of this width")
a = ap.parse_args()
A = S.laplacian_3d(a.grid)
f = S.ilu_k(A, 0)
ML = S.sait_thr(S.DeviceCsr.upload(f.lower), S.lower_triangular, S.SaitThrParams(5e-2, 3))
MU = S.sait_thr(S.DeviceCsr.upload(f.upper), S.upper_triangular, S.SaitThrParams(5e-2, 3))
pair = S.SaitPairPreconditioner(ML, MU)
r = torch.from_numpy(S.uniform_pm1(1000, A.nrows)).cuda()
z = torch.empty_like(r)
for _ in range(a.applies):
    pair.apply(r, z)
if a.block:
    R = torch.rand((A.nrows, a.block), dtype=torch.float64, device="cuda")
    for _ in range(a.applies):
        pair.apply_block(R, layout="row")
torch.cuda.synchronize()
print("ok", ML.nnz(), MU.nnz())
