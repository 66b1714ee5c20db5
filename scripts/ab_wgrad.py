"""Weight-gradient GEMM tile shapes on the configs[1] shapes (tokens 18432):
1-SM 128-row vs 2-SM 256-row tiles x BN 128 / 256, plus auto; interleaved
rounds, median TFLOP/s (useful flops)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_05019_b200 import kernels as K
T = 18432
shapes = [("w1 1536x384", 1536, 384), ("w2 384x1536", 384, 1536), ("qkv 1152x384", 1152, 384),
          ("o 384x384", 384, 384)]
if len(sys.argv) > 1 and sys.argv[1] == "moe":    # 16 experts x 1440 rows
    T = None
res = {}
for name, M, N in shapes:
    a = torch.randn(1, T, M, device="cuda").bfloat16()
    b = torch.randn(1, T, N, device="cuda").bfloat16()
    def arm(mode, bn, flags=0):
        def f():
            K.set_gemm_mode(mode)
            K.set_gemm_tile_n(bn)
            K.set_gemm_flags(flags)
            K.grouped_wgrad(a, b, n_wgroups=1)
            K.set_gemm_flags(0)
        return f
    # *_rowst: the row-per-thread fp32 partial stores (flag 16) instead of staged
    arms = {"auto": arm(0, 0), "auto_rowst": arm(0, 0, 16), "1sm128": arm(1, 128),
            "1sm256": arm(1, 256), "2sm128": arm(2, 128), "2sm256": arm(2, 256),
            "2sm256_rowst": arm(2, 256, 16)}
    for _ in range(3):
        for f in arms.values(): f()
    for r in range(5):
        for key, f in arms.items():
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20): f()
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            res.setdefault((name, key), []).append(2 * T * M * N / ms / 1e9)
K.set_gemm_mode(0); K.set_gemm_tile_n(0)
for (name, key), v in res.items():
    print(f"{name:14s} {key:7s} {statistics.median(v):7.0f} TFLOP/s")
