import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_05019_b200 import kernels as K
for kd in (64, 128, 200):
    a = torch.randn(256, kd, device="cuda").bfloat16()
    bad = []
    for n in range(8, 400, 8):
        w = torch.randn(n, kd, device="cuda").bfloat16()
        ref = (a.float() @ w.float().t())
        for mode in (1, 2):
            K.set_gemm_mode(mode); K.set_gemm_tile_n(192)
            o = K.grouped_gemm(a, w, None).float()
            torch.cuda.synchronize()
            err = float((o - ref).abs().max() / ref.abs().max())
            if err > 1e-2:
                bad.append((n, mode, round(err, 3)))
    print("K", kd, "bad", bad)
K.set_gemm_mode(0); K.set_gemm_tile_n(0)
