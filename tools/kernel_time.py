"""Device time per kernel name of one capped config-4 build with k recursion
steps (torch.profiler), for kernel A/B variants (SAIT_LIB_VARIANT):
python tools/kernel_time.py [log2 n] [k] [name-regex]"""
import os
import re
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12836_b200 as S  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pat = re.compile(sys.argv[3] if len(sys.argv) > 3 else ".")
T = S.DeviceCsr.upload(S.synthetic_lower(1 << lg, 15, 0.01, 4))
S.reserve_device_pool(40 << 30)


def run():
    m = S.sait_thr_cap(T, S.lower_triangular, S.SaitThrParams(1e-2, k), 3.0)
    torch.cuda.synchronize()
    m.free()


for _ in range(2):
    run()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
per = defaultdict(list)
for e in prof.events():
    if e.device_type != torch.autograd.DeviceType.CUDA:
        continue
    name = re.sub(r"\(anonymous namespace\)::|^void ", "", e.name).split("(")[0]
    if pat.search(name):
        per[name].append((e.time_range.end - e.time_range.start) / 1e3)
tag = os.environ.get("SAIT_LIB_VARIANT", "default")
for name, ts in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    print(f"{tag:10s} {sum(ts):8.3f} ms  {name}  per launch {[round(t, 3) for t in ts]}")
