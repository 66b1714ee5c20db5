"""ncu target: one configs[1] training GEMM shape, with / without residual.
python scripts/gemm_one.py K N layout(nk|kn) res(0|1) [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2404_05019_b200 import _lib as L
from paper_2404_05019_b200 import kernels as K

Kd, N = int(sys.argv[1]), int(sys.argv[2])
lay = L.W_NK if sys.argv[3] == "nk" else L.W_KN
res = sys.argv[4] == "1"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
M = 18432
a = torch.randn(M, Kd, device="cuda").bfloat16()
w = (torch.randn(N, Kd, device="cuda") / Kd ** 0.5).bfloat16()
if lay == L.W_KN:
    w = w.t().contiguous()
r = torch.randn(M, N, device="cuda").bfloat16() if res else None
for _ in range(reps):
    K.grouped_gemm_ex(a, w, lay, N, residual=r)
torch.cuda.synchronize()
