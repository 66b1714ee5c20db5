"""Each GEMM call of the configs[1] training step (training.py LinearFn /
FFNFn, T = 18432, d = 384, h = 1536) timed alone with its real epilogue:
useful TFLOP/s and the output-side bytes, to find the weak calls."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_05019_b200 import kernels as K, _lib as L
T, d, h = 18432, 384, 1536
bf = dict(device="cuda", dtype=torch.bfloat16)
x = torch.randn(T, d, **bf); res = torch.randn(T, d, **bf)
wqkv = torch.randn(3 * d, d, **bf) / 20; wo = torch.randn(d, d, **bf) / 20
w1 = torch.randn(1, h, d, **bf) / 20; w2 = torch.randn(1, d, h, **bf) / 20
b1 = torch.zeros(1, h, device="cuda"); b2 = torch.zeros(1, d, device="cuda")
z = torch.empty(1, T, h, **bf); hid = torch.randn(1, T, h, **bf)
dy = torch.randn(1, T, d, **bf); dqkv = torch.randn(T, 3 * d, **bf)
rows = torch.tensor([T], device="cuda", dtype=torch.int32)
x3, res3 = x.view(1, T, d), res.view(1, T, d)
calls = {
    "qkv fwd": (lambda: K.grouped_gemm(x, wqkv, None), 2 * T * d * 3 * d),
    "o fwd +res": (lambda: K.grouped_gemm(x, wo, None, residual=res), 2 * T * d * d),
    "ffn1 fwd b+gelu+z": (lambda: K.grouped_gemm_ex(x3, w1, L.W_NK, h, bias=b1, aux_out=z,
                                                   epilogue=L.EPI_BIAS_GELU), 2 * T * d * h),
    "ffn1 fwd b+gelu": (lambda: K.grouped_gemm_ex(x3, w1, L.W_NK, h, bias=b1,
                                                 epilogue=L.EPI_BIAS_GELU), 2 * T * d * h),
    "ffn2 fwd b+res": (lambda: K.grouped_gemm_ex(hid, w2, L.W_NK, d, bias=b2, residual=res3),
                       2 * T * d * h),
    "ffn2 dgrad gelu'": (lambda: K.grouped_gemm_ex(dy, w2, L.W_KN, h, aux_in=z,
                                                  epilogue=L.EPI_GELU_BWD, group_rows=rows,
                                                  rows_clip=T, zero_tail=True), 2 * T * d * h),
    "ffn2 dgrad plain": (lambda: K.grouped_gemm_ex(dy, w2, L.W_KN, h), 2 * T * d * h),
    "ffn1 dgrad": (lambda: K.grouped_gemm_ex(hid, w1, L.W_KN, d, group_rows=rows, rows_clip=T),
                   2 * T * d * h),
    "qkv dgrad": (lambda: K.grouped_gemm_ex(dqkv, wqkv, L.W_KN, d), 2 * T * d * 3 * d),
    "o dgrad": (lambda: K.grouped_gemm_ex(x, wo, L.W_KN, d), 2 * T * d * d),
    "bias grad h": (lambda: K.bias_grad(hid), 2 * T * h * 8),
    "colsum h": (lambda: K.grouped_colsum(hid, rows, T), 2 * T * h * 8),
    "bias grad d": (lambda: K.bias_grad(dy), 2 * T * d * 8),
    "colsum d": (lambda: K.grouped_colsum(dy, rows, T), 2 * T * d * 8),
}
res_t = {}
for _ in range(3):
    for f, _fl in calls.values(): f()
for r in range(5):
    for name, (f, fl) in calls.items():
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        res_t.setdefault(name, []).append((e0.elapsed_time(e1) / 20, fl))
for name, v in res_t.items():
    ms = statistics.median(t for t, _ in v)
    print(f"{name:20s} {ms * 1e3:8.1f} us {v[0][1] / ms / 1e9:7.0f} TFLOP/s")
