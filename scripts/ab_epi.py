"""A/B of the GEMM epilogue width (8 vs 16 epilogue warps) on the configs[1]
training GEMM calls and the configs[2] forward GEMMs, interleaved rounds.

    python scripts/ab_epi.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_05019_b200 import kernels as K, _lib as L

bf = dict(device="cuda", dtype=torch.bfloat16)


def calls_for(T, d, h):
    x = torch.randn(T, d, **bf)
    res = torch.randn(T, d, **bf)
    w1 = torch.randn(1, h, d, **bf) / 20
    w2 = torch.randn(1, d, h, **bf) / 20
    b1 = torch.zeros(1, h, device="cuda")
    b2 = torch.zeros(1, d, device="cuda")
    z = torch.empty(1, T, h, **bf)
    hid = torch.randn(1, T, h, **bf)
    dy = torch.randn(1, T, d, **bf)
    wo = torch.randn(d, d, **bf) / 20
    rows = torch.tensor([T], device="cuda", dtype=torch.int32)
    x3, res3 = x.view(1, T, d), res.view(1, T, d)
    fl = 2 * T * d * h
    return {
        f"ffn1 b+gelu+z {d}": (lambda: K.grouped_gemm_ex(x3, w1, L.W_NK, h, bias=b1, aux_out=z,
                                                        epilogue=L.EPI_BIAS_GELU), fl),
        f"ffn1 b+gelu {d}": (lambda: K.grouped_gemm_ex(x3, w1, L.W_NK, h, bias=b1,
                                                      epilogue=L.EPI_BIAS_GELU), fl),
        f"ffn2 b+res {d}": (lambda: K.grouped_gemm_ex(hid, w2, L.W_NK, d, bias=b2, residual=res3),
                            fl),
        f"ffn2 dgrad gelu' {d}": (lambda: K.grouped_gemm_ex(dy, w2, L.W_KN, h, aux_in=z,
                                                           epilogue=L.EPI_GELU_BWD, group_rows=rows,
                                                           rows_clip=T, zero_tail=True), fl),
        f"o fwd +res {d}": (lambda: K.grouped_gemm(x, wo, None, residual=res), 2 * T * d * d),
    }


calls = calls_for(18432, 384, 1536)
calls.update(calls_for(16384, 2048, 8192))
res = {}
for _ in range(2):
    for f, _fl in calls.values():
        f()
for r in range(5):
    for epi in (8, 16):
        K.set_gemm_epilogue_warps(epi)
        for name, (f, fl) in calls.items():
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                f()
            e1.record()
            torch.cuda.synchronize()
            res.setdefault((name, epi), []).append((e0.elapsed_time(e1) / 10, fl))
K.set_gemm_epilogue_warps(0)
for name in calls:
    row = []
    for epi in (8, 16):
        v = res[(name, epi)]
        ms = statistics.median(t for t, _ in v)
        row.append(f"E{epi}: {ms * 1e3:7.1f} us {v[0][1] / ms / 1e9:6.0f} TF/s")
    print(f"{name:28s} " + " | ".join(row))
