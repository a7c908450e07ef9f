"""Times the block-8 pair apply (column-major n x 8 device block, LOBPCG's
M R) on config 5's factors (or grid^3): ms per block and the format-byte
rate.  For block-kernel experiments.  python tools/block_time.py [grid=256]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_12836_b200 as S  # noqa: E402

grid = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = S.laplacian_3d(grid)
dA = S.DeviceCsr.upload(A)
f = S.ilu0_device(dA)
ML, MU = S.sait_thr_pair(f.lower, f.upper, S.SaitThrParams(5e-2, 3))
pair = S.SaitPairPreconditioner(ML, MU)
n = A.nrows
R = torch.rand((8, n), dtype=torch.float64, device="cuda")
Z = torch.empty_like(R)
for _ in range(3):
    pair.apply_block(R.T, Z.T)
torch.cuda.synchronize()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        pair.apply_block(R.T, Z.T)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 5)
ms = sorted(ts)[3]
fb = sum(pair.factor_format(w)["stream_bytes"] for w in (0, 1)) + 2 * 14 * 8 * n
print(f"grid={grid} ms_per_block8={ms:.4f} "
      f"format_TBs={fb / ms / 1e9:.3f} checksum={float(Z.sum()):.17g}")
