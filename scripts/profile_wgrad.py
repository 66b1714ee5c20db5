"""ncu target: the configs[1] FFN1 weight gradient (dW1 = dz^T x over 18432
tokens, 1536 x 384) with the tile mode from argv[1] (0 auto, 1 1-SM, 2 2-SM)
and BN from argv[2]; 3 calls (capture the last with -s 2 -c 1 on
regex:gemm_kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_05019_b200 import kernels as K
T, M, N = 18432, 1536, 384
a = torch.randn(1, T, M, device="cuda").bfloat16()
b = torch.randn(1, T, N, device="cuda").bfloat16()
K.set_gemm_mode(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
K.set_gemm_tile_n(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
for _ in range(3):
    K.grouped_wgrad(a, b, n_wgroups=1)
torch.cuda.synchronize()
