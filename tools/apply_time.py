"""Times the C2 (or C5) pair step the way bench.py does (100 sequential pair
applies on distinct device vectors, CUDA events, 3 repeats) -- for kernel
experiments selected by environment variables.  Prints ms per step and the
per-launch time.  python tools/apply_time.py [grid=128] [format=auto]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_12836_b200 as S  # noqa: E402

grid = int(sys.argv[1]) if len(sys.argv) > 1 else 128
fmt = sys.argv[2] if len(sys.argv) > 2 else "auto"
nvec = 100 if grid <= 128 else 20
A = S.laplacian_3d(grid)
dA = S.DeviceCsr.upload(A)
f = S.ilu0_device(dA)
ML, MU = S.sait_thr_pair(f.lower, f.upper, S.SaitThrParams(5e-2, 3))
pair = S.SaitPairPreconditioner(ML, MU, format=fmt)
n = A.nrows
R = torch.empty((nvec, n), dtype=torch.float64, device="cuda")
for i in range(nvec):
    R[i].copy_(torch.from_numpy(S.uniform_pm1(1000 + i, n)))
Z = torch.empty_like(R)
ref = None


def step():
    for i in range(nvec):
        pair.apply(R[i], Z[i])


for _ in range(3):
    step()
torch.cuda.synchronize()
out = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step()
    e1.record()
    torch.cuda.synchronize()
    out.append(e0.elapsed_time(e1))
ms = sorted(out)[2]
fb = pair.factor_format(0)["stream_bytes"] + pair.factor_format(1)["stream_bytes"]
print(f"grid={grid} fmt={fmt} lib={os.environ.get('SAIT_LIB_VARIANT', 'default')} ms_per_step={ms:.4f} "
      f"us_per_launch={1e3 * ms / (2 * nvec):.2f} format_TBs={nvec * fb / ms / 1e9:.3f} checksum={float(Z.sum()):.17g}")
