"""Times the SAIT pair of config 4's T and T^T (n = 2^lg; the non-stencil
pattern) as bench.py's build_c4.irregular_apply does: 20 sequential pair
applies on device vectors, CUDA events.  python tools/irregular_apply.py [lg]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_12836_b200 as S  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
T = S.DeviceCsr.upload(S.synthetic_lower(1 << lg, 15, 0.01, 4))
P = S.SaitThrParams(1e-2, 3)
ML = S.sait_thr(T, S.lower_triangular, P)
MU = S.sait_thr(S.transpose(T), S.upper_triangular, P)
pair = S.SaitPairPreconditioner(ML, MU)
n = ML.nrows
R = torch.empty((20, n), dtype=torch.float64, device="cuda")
for i in range(20):
    R[i].copy_(torch.from_numpy(S.uniform_pm1(7000 + i, n)))
Z = torch.empty_like(R)


def step():
    for i in range(20):
        pair.apply(R[i], Z[i])


for _ in range(3):
    step()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[2]
fb = pair.factor_format(0)["stream_bytes"] + pair.factor_format(1)["stream_bytes"]
print({"formats": [pair.factor_format(w)["format"] + ("+sorted" if pair.factor_format(w)["row_sorted"] else "")
                   for w in (0, 1)], "ms_per_pair": ms / 20, "format_TBs": 20 * fb / ms / 1e9,
       "frac_of_6548_GBs": 20 * fb / ms / 1e9 / 6.5485, "checksum": float(Z.sum())})
