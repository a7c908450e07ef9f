import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2106_12836_b200 as S
g = int(sys.argv[1])
A = S.laplacian_3d(g)
f = S.ilu0_device(A)
P = S.SaitPairPreconditioner(S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3)), S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(5e-2, 3)))
n = A.nrows
R = torch.rand((8, n), dtype=torch.float64, device="cuda")  # column-major n x 8 (rows of this = columns)
Z = torch.empty_like(R)
from paper_2106_12836_b200 import _native as N
s = torch.cuda.current_stream().cuda_stream
def run():
    N.check(N.lib.sait_pair_apply_block(P.handle, R.data_ptr(), Z.data_ptr(), n, 8, 0, s))
for _ in range(3): run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): run()
b.record(); torch.cuda.synchronize()
print(os.environ.get("SAIT_BLOCK_CM", "1"), g, "ms per block-8 apply", a.elapsed_time(b) / 10)
