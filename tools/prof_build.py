"""C2 factor builds only (for ncu on the builder kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12836_b200 as S
A = S.laplacian_3d(int(sys.argv[1]) if len(sys.argv) > 1 else 128)
f = S.ilu_k(A, 0)
L = S.DeviceCsr.upload(f.lower)
for _ in range(2):
    st = []
    M = S.sait_thr(L, S.lower_triangular, S.SaitThrParams(5e-2, 3), stats_out=st)
    print(st[0])
torch.cuda.synchronize()
