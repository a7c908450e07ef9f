"""Per-kernel device time of one SAIT build (torch.profiler / CUPTI).

python tools/build_breakdown.py c2      # pair build of the C2 factors (bench)
python tools/build_breakdown.py c4 [lg] # capped C4 build (BASELINE config 4)

Prints the span, the summed kernel time per kernel name, and the idle time
(no kernel or copy running) — where a build's wall time goes."""
import os
import re
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12836_b200 as S  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
if which == "c2":
    A = S.laplacian_3d(128)
    f = S.ilu_device(A, 0)
    P = S.SaitThrParams(5e-2, 3)
    S.reserve_device_pool(4 << 30)

    def run():
        a, b = S.sait_thr_pair(f.lower, f.upper, P)
        torch.cuda.synchronize()
        a.free()
        b.free()
else:
    lg = int(sys.argv[2]) if len(sys.argv) > 2 else 24
    T = S.DeviceCsr.upload(S.synthetic_lower(1 << lg, 15, 0.01, 4))
    S.reserve_device_pool(40 << 30)

    def run():
        m = S.sait_thr_cap(T, S.lower_triangular, S.SaitThrParams(1e-2, 3), 3.0)
        torch.cuda.synchronize()
        m.free()

for _ in range(3):
    run()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in ev)
t1 = max(e.time_range.end for e in ev)
per = defaultdict(lambda: [0, 0.0])
for e in ev:
    k = re.sub(r"\(anonymous namespace\)::", "", e.name)
    k = re.sub(r"^void ", "", k)
    k = k.split("(")[0][:60]
    per[k][0] += 1
    per[k][1] += e.time_range.end - e.time_range.start
iv = sorted((e.time_range.start, e.time_range.end) for e in ev)
covered, cs, ce = 0.0, iv[0][0], iv[0][1]
for s, e in iv[1:]:
    if s > ce:
        covered += ce - cs
        cs, ce = s, e
    else:
        ce = max(ce, e)
covered += ce - cs
print(f"{which}: span {(t1 - t0) / 1e3:.3f} ms, device busy {covered / 1e3:.3f} ms, idle {(t1 - t0 - covered) / 1e3:.3f} ms")
for k, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
    print(f"  {t / 1e3:8.3f} ms  {c:4d}x  {k}")
