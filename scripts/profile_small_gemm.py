"""ncu target: configs[1] FFN GEMM1 shape (18432 x 384 -> 1536), plain store
(argv[1] == "plain", default) or bias + GELU ("gelu")."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_05019_b200 import kernels as K
M, Kd, N = 18432, 384, 1536
a = torch.randn(M, Kd, device="cuda").bfloat16()
wt = (torch.randn(N, Kd, device="cuda") / Kd ** 0.5).bfloat16()
b = torch.zeros(N, device="cuda")
gelu = len(sys.argv) > 1 and sys.argv[1] == "gelu"
for _ in range(4):
    K.grouped_gemm(a, wt, b if gelu else None, gelu=gelu)
torch.cuda.synchronize()
