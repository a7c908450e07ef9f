"""Short C2 apply driver for ncu (not a benchmark: nothing is timed).

Builds the config-2 pair on the device, then runs `--pairs` applies
z_i = M_U (M_L r_i) back to back on DISTINCT seeded vectors -- the timed
condition of bench.py -- in the requested apply format.  Profile with
  ncu --cache-control none --clock-control none -k regex:sell_spmv|spmv_tma \\
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \\
      --csv --log-file out.csv python tools/ncu_apply.py
so the L2 state one launch leaves is what the next one sees, then summarise
with tools/ncu_traffic.py."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_12836_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=128)
ap.add_argument("--pairs", type=int, default=8)
ap.add_argument("--format", default="auto")
a = ap.parse_args()
A = S.laplacian_3d(a.grid)
f = S.ilu_k(A, 0)
ML, MU = S.sait_thr_pair(S.DeviceCsr.upload(f.lower), S.DeviceCsr.upload(f.upper), S.SaitThrParams(5e-2, 3))
pair = S.SaitPairPreconditioner(ML, MU, format=a.format)
n = A.nrows
R = torch.empty((a.pairs, n), dtype=torch.float64, device="cuda")
for i in range(a.pairs):
    R[i].copy_(torch.from_numpy(S.uniform_pm1(1000 + i, n)))
Z = torch.empty_like(R)
for i in range(a.pairs):
    pair.apply(R[i], Z[i])
torch.cuda.synchronize()
print("ok", a.format, pair.factor_format(0)["format"], pair.factor_format(1)["format"],
      pair.factor_format(0)["stream_bytes"], pair.factor_format(1)["stream_bytes"])
