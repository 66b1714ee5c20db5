"""Our tcgen05 GEMM vs cuBLAS (torch.matmul) on the configs[2] dense shapes,
interleaved rounds (power-cap drift hits both), median TFLOP/s."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_05019_b200 import kernels as K
shapes = [("ffn1 16384x2048->8192", 16384, 2048, 8192), ("ffn2 16384x8192->2048", 16384, 8192, 2048),
          ("qkv 16384x2048->6144", 16384, 2048, 6144)]
if len(sys.argv) > 1 and sys.argv[1] == "train":      # configs[1] (d 384, h 1536) shapes
    shapes = [("ffn1 18432x384->1536", 18432, 384, 1536), ("ffn2 18432x1536->384", 18432, 1536, 384),
              ("qkv 18432x384->1152", 18432, 384, 1152), ("o 18432x384->384", 18432, 384, 384)]
res = {}
for name, M, Kd, N in shapes:
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    wt = (torch.randn(N, Kd, device="cuda") / Kd ** 0.5).bfloat16()
    w = wt.t().contiguous()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    def ours(bn):
        def f():
            K.set_gemm_tile_n(bn)
            K.grouped_gemm(a, wt, None, out=out)
        return f
    fns = {"ours": ours(0), "ours256": ours(256), "cublas": lambda: torch.matmul(a, w, out=out)}
    for _ in range(3):
        for f in fns.values(): f()
    for r in range(6):
        for key, f in fns.items():
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20): f()
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            res.setdefault((name, key), []).append(2 * M * Kd * N / ms / 1e9)
for (name, key), v in res.items():
    print(f"{name:24s} {key:7s} {statistics.median(v):7.0f} TFLOP/s")
