"""Tile-shape sweep of our tcgen05 GEMM on the configs[1] training shapes vs
cuBLAS: 1-SM / 2-SM, BN 128 / 192 / 256, auto epilogue warps; us per call
as 20 back-to-back launches (PDL chains them, as in the step), interleaved
rounds, medians.

    python scripts/sweep_small_gemm.py
"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_05019_b200 import kernels as K

shapes = [("ffn1 18432x384->1536", 18432, 384, 1536, False),
          ("ffn2+res 18432x1536->384", 18432, 1536, 384, True),
          ("qkv 18432x384->1152", 18432, 384, 1152, False),
          ("o+res 18432x384->384", 18432, 384, 384, True)]
res = {}
for name, M, Kd, N, resid in shapes:
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    wt = (torch.randn(N, Kd, device="cuda") / Kd ** 0.5).bfloat16()
    w = wt.t().contiguous()
    r = torch.randn(M, N, device="cuda").bfloat16() if resid else None
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)

    def ours(mode, bn):
        def f():
            K.set_gemm_mode(mode)
            K.set_gemm_tile_n(bn)
            K.grouped_gemm(a, wt, None, out=out, residual=r)
        return f
    fns = {}
    for mode in (0, 1, 2):
        for bn in (0, 128, 192, 256):
            if mode == 0 and bn:
                continue
            fns[f"m{mode}bn{bn}"] = ours(mode, bn)
    if resid:
        fns["cublas"] = lambda: torch.addmm(r, a, w, out=out)
    else:
        fns["cublas"] = lambda: torch.matmul(a, w, out=out)
    for _ in range(3):
        for f in fns.values():
            f()
    for rnd in range(5):
        for key, f in fns.items():
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                f()
            e1.record()
            torch.cuda.synchronize()
            res.setdefault((name, key), []).append(e0.elapsed_time(e1) / 20 * 1e3)
    K.set_gemm_mode(0)
    K.set_gemm_tile_n(0)
for name, *_ in shapes:
    line = [f"{k}={statistics.median(v):.1f}" for (n, k), v in res.items() if n == name]
    print(f"{name:26s} us: " + " ".join(line))
