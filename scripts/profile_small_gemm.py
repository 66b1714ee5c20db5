"""ncu target: configs[1] FFN GEMM1 shape (18432 x 384 -> 1536), plain store
(argv[1] == "plain", default), bias + GELU ("gelu"), or the GELU-backward
dgrad ("gbwd")."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_05019_b200 import kernels as K
M, Kd, N = 18432, 384, 1536
a = torch.randn(M, Kd, device="cuda").bfloat16()
wt = (torch.randn(N, Kd, device="cuda") / Kd ** 0.5).bfloat16()
b = torch.zeros(N, device="cuda")
mode = sys.argv[1] if len(sys.argv) > 1 else "plain"
K.set_gemm_epilogue_warps(int(os.environ.get("SCMOE_EPI", "0")))
gelu = mode == "gelu"
if mode == "gbwd":        # training dgrad: dZ = (dY . W2) * gelu'(z), configs[1] shape
    from paper_2404_05019_b200 import _lib as L
    dy = torch.randn(1, M, Kd, device="cuda").bfloat16()
    w2 = (torch.randn(1, Kd, N, device="cuda") / 20).bfloat16()
    z = torch.randn(1, M, N, device="cuda").bfloat16()
    rows = torch.tensor([M], device="cuda", dtype=torch.int32)
    fn = lambda: K.grouped_gemm_ex(dy, w2, L.W_KN, N, aux_in=z, epilogue=L.EPI_GELU_BWD,
                                   group_rows=rows, rows_clip=M, zero_tail=True)
else:
    fn = lambda: K.grouped_gemm(a, wt, b if gelu else None, gelu=gelu)
for _ in range(4):
    fn()
torch.cuda.synchronize()
