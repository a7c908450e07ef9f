"""Does sait_build_pair overlap the two recursions?  Kernel intervals per
stream from one profiled pair build (torch.profiler / CUPTI)."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12836_b200 as S  # noqa: E402

A = S.laplacian_3d(128)
f = S.ilu_device(A, 0)
L, U = f.lower, f.upper
P = S.SaitThrParams(5e-2, 3)
S.reserve_device_pool(4 << 30)
for _ in range(3):
    a, b = S.sait_thr_pair(L, U, P)
    a.free()
    b.free()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    a, b = S.sait_thr_pair(L, U, P)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
streams = {}
for e in ev:
    sid = getattr(e, "stream", None)
    if sid is None:
        sid = e.device_resource_id if hasattr(e, "device_resource_id") else 0
    streams.setdefault(sid, []).append((e.time_range.start, e.time_range.end, e.name[:40]))
t0 = min(e.time_range.start for e in ev)
t1 = max(e.time_range.end for e in ev)
print(f"span {(t1 - t0) / 1e3:.3f} ms, streams {len(streams)}")
busy = {}
for sid, iv in streams.items():
    iv.sort()
    b = sum(e - s for s, e, _ in iv)
    busy[sid] = b
    print(f"stream {sid}: {len(iv)} ops, busy {b / 1e3:.3f} ms, first {(iv[0][0] - t0) / 1e3:.3f} last {(iv[-1][1] - t0) / 1e3:.3f}")
# overlap: time covered by >= 2 streams
pts = []
for sid, iv in streams.items():
    for s, e, _ in iv:
        pts.append((s, 1))
        pts.append((e, -1))
pts.sort()
cur, last, both, any_ = 0, None, 0.0, 0.0
for t, d in pts:
    if last is not None:
        if cur >= 2:
            both += t - last
        if cur >= 1:
            any_ += t - last
    cur += d
    last = t
print(f"covered {any_ / 1e3:.3f} ms, by >= 2 streams {both / 1e3:.3f} ms")
# idle intervals (no stream busy), with the op that ends before and starts after
allv = sorted((s, e, n, sid) for sid, iv in streams.items() for s, e, n in iv)
gaps = []
end, endname = allv[0][1], allv[0][2]
for s, e, n, sid in allv[1:]:
    if s > end:
        gaps.append((s - end, endname, n))
    if e > end:
        end, endname = e, n
gaps.sort(reverse=True)
print(f"idle {sum(g for g, _, _ in gaps) / 1e3:.3f} ms in {len(gaps)} gaps; largest:")
for g, a, b in gaps[:14]:
    print(f"  {g:7.1f} us  after {a:40s} before {b}")
