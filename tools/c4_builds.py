"""Repeated C4 builds (BASELINE config 4, capped): seconds per build as the
library measures it.  python tools/c4_builds.py [log2 n] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_12836_b200 as S  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
T = S.DeviceCsr.upload(S.synthetic_lower(1 << lg, 15, 0.01, 4))
S.reserve_device_pool(int(float(os.environ.get("SAIT_C4_RESERVE_GB", "40")) * (1 << 30)))  # no pool growth in the timings
out = []
for _ in range(reps):
    st = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = S.sait_thr_cap(T, S.lower_triangular, S.SaitThrParams(1e-2, 3), 3.0, stats_out=st)
    torch.cuda.synchronize()
    out.append((round(st[0].seconds, 4), round(time.perf_counter() - t0, 4)))
    m.free()
print("builds (device s, wall s):", out)
