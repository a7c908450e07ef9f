"""Kernel timeline of one C2 factor build (or pair apply, or 5 LOBPCG iterations) via torch.profiler
(CUPTI): per-kernel device time, the busy fraction of the wall interval and
the largest idle gaps.  python tools/prof_timeline.py [build|pair|apply|lobpcg|ilu0|ilu1|c4] [grid]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2106_12836_b200 as S  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "build"
grid = int(sys.argv[2]) if len(sys.argv) > 2 else 128
if what == "c4":  # BASELINE config 4 build (grid = log2 n, default 24)
    T = S.DeviceCsr.upload(S.synthetic_lower(1 << (grid if grid < 64 else 24), 15, 0.01, 4))
    A = None
else:
    A = S.laplacian_3d(grid)
    f = S.ilu_k(A, 0)
    L = S.DeviceCsr.upload(f.lower)
    U = S.DeviceCsr.upload(f.upper)


def build():
    S.sait_thr(L, S.lower_triangular, S.SaitThrParams(5e-2, 3))
    S.sait_thr(U, S.upper_triangular, S.SaitThrParams(5e-2, 3))


run = build
if what == "pair":  # both factors through sait_build_pair (concurrent recursions)
    def run():
        a, b = S.sait_thr_pair(L, U, S.SaitThrParams(5e-2, 3))
        a.free()
        b.free()
if what in ("ilu0", "ilu1"):
    dA = S.DeviceCsr.upload(A)

    def run():
        g = S.ilu_device(dA, int(what[-1]))
        g.lower.free()
        g.upper.free()
if what == "c4":
    def run():
        m = S.sait_thr_cap(T, S.lower_triangular, S.SaitThrParams(1e-2, 3), 3.0)
        m.free()
if what == "lobpcg":
    ML = S.sait_thr(L, S.lower_triangular, S.SaitThrParams(5e-2, 3))
    MU = S.sait_thr(U, S.upper_triangular, S.SaitThrParams(5e-2, 3))
    P = S.SaitPairPreconditioner(ML, MU)
    dA = S.DeviceCsr.upload(A)

    def run():
        S.lobpcg(dA, P, 8, 1e-6, 5, 5, host_vectors=False, gram=os.environ.get("SAIT_LOBPCG_GRAM", "canonical"))
if what == "apply":
    ML = S.sait_thr(L, S.lower_triangular, S.SaitThrParams(5e-2, 3))
    MU = S.sait_thr(U, S.upper_triangular, S.SaitThrParams(5e-2, 3))
    P = S.SaitPairPreconditioner(ML, MU)
    r = torch.rand(A.nrows, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)

    def run():
        for _ in range(10):
            P.apply(r, z)

for _ in range(2):
    run()
torch.cuda.synchronize()
t0 = time.perf_counter()
run()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    run()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t_first, t_last = ev[0].time_range.start, max(e.time_range.end for e in ev)
busy = sum(e.time_range.elapsed_us() for e in ev)
print(f"{what}: wall {wall:.3f} ms (unprofiled); device span {(t_last - t_first) / 1e3:.3f} ms, busy {busy / 1e3:.3f} ms, {len(ev)} device ops")
agg = {}
for e in ev:
    k = e.name[:80]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += e.time_range.elapsed_us()
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:18]:
    print(f"{t / 1e3:8.3f} ms {c:4d}x  {k}")
gaps = []
end = ev[0].time_range.end
for e in ev[1:]:
    if e.time_range.start > end:
        gaps.append((e.time_range.start - end, e.name[:60]))
    end = max(end, e.time_range.end)
gaps.sort(reverse=True)
print("idle total %.3f ms; largest gaps (us, before):" % (sum(g for g, _ in gaps) / 1e3), [(round(g, 1), n) for g, n in gaps[:10]])
