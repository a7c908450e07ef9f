"""Host-vector apply (e2e path) probe at BASELINE config 2: ms per apply for
several chunk schedules (SAIT_PIPE_MB), plus one debug timeline
(SAIT_DEBUG_PIPE) and the raw PCIe copy times of r and z.

    python tools/e2e_probe.py [schedule ...]
"""
import os
import subprocess
import sys
import time

if os.environ.get("_E2E_CHILD"):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch

    import paper_2106_12836_b200 as S

    A = S.laplacian_3d(128)
    f = S.ilu_k(A, 0)
    ML = S.sait_thr(S.DeviceCsr.upload(f.lower), S.lower_triangular, S.SaitThrParams(5e-2, 3))
    MU = S.sait_thr(S.DeviceCsr.upload(f.upper), S.upper_triangular, S.SaitThrParams(5e-2, 3))
    pair = S.SaitPairPreconditioner(ML, MU)
    n = A.nrows
    r = torch.from_numpy(S.uniform_pm1(1, n)).pin_memory()
    z = torch.empty_like(r).pin_memory()
    for _ in range(5):
        pair.apply(r.numpy(), z.numpy())
    reps = 50
    t0 = time.perf_counter()
    for _ in range(reps):
        pair.apply(r.numpy(), z.numpy())
    ms = (time.perf_counter() - t0) / reps * 1e3
    print(f"schedule={os.environ.get('SAIT_PIPE_MB', 'default')} ms_per_apply={ms:.4f} e2e_GBs={432677896 / ms / 1e6:.1f}")
    if os.environ.get("_E2E_RAW"):
        rd = torch.empty(n, dtype=torch.float64, device="cuda")
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        torch.cuda.synchronize()

        def t(fn, k=20):
            fn()
            torch.cuda.synchronize()
            a = time.perf_counter()
            for _ in range(k):
                fn()
            torch.cuda.synchronize()
            return (time.perf_counter() - a) / k * 1e3

        h2d = t(lambda: rd.copy_(r, non_blocking=True))
        d2h = t(lambda: z.copy_(rd, non_blocking=True))

        def both():
            with torch.cuda.stream(s1):
                rd.copy_(r, non_blocking=True)
            with torch.cuda.stream(s2):
                z.copy_(rd2, non_blocking=True)

        rd2 = torch.empty_like(rd)
        bb = t(both)
        print(f"raw: h2d {h2d:.4f} ms ({8 * n / h2d / 1e6:.1f} GB/s)  d2h {d2h:.4f} ms ({8 * n / d2h / 1e6:.1f} GB/s)  both {bb:.4f} ms")
    if os.environ.get("SAIT_DEBUG_PIPE"):
        pass
    sys.exit(0)

scheds = sys.argv[1:] or ["default", "1", "2", "4", "8", "1,2,4", "2,4,1", "4,4,2", "2,2,1", "zc0:2,4,1"]
for i, sc in enumerate(scheds):
    env = dict(os.environ, _E2E_CHILD="1")
    if sc.startswith("zc0:"):
        env["SAIT_HOST_ZC_OUT"] = "0"
        sc = sc[4:]
    if sc != "default":
        env["SAIT_PIPE_MB"] = sc
    if i == 0:
        env["_E2E_RAW"] = "1"
    out = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
    print(out.stdout.strip(), out.stderr.strip()[-300:] if out.returncode else "")
env = dict(os.environ, _E2E_CHILD="1", SAIT_DEBUG_PIPE="1")
out = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
print("timeline (us since enqueue start), last apply:")
print(out.stderr.strip().splitlines()[-1] if out.stderr.strip() else out.stdout)
