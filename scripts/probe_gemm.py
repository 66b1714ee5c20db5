"""Quick device-time probe of the hot kernels at the configs[2] shape
(T=16384, d=2048, h=8192, N=8, cf=2.0) vs cuBLAS (torch.matmul)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_05019_b200 import kernels as K


def t_ms(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    T, d, h, N = 16384, 2048, 8192, 8
    res = {}
    x = torch.randn(T, d, device="cuda").bfloat16()
    w1t = (torch.randn(h, d, device="cuda") / d ** 0.5).bfloat16()
    b1 = torch.zeros(h, device="cuda")
    out = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
    for mode in (1, 2):
        K.set_gemm_mode(mode)
        ms = t_ms(lambda: K.grouped_gemm(x, w1t, b1, gelu=True, out=out))
        res[f"mode{mode}_dense_gemm1_gelu_tflops"] = 2 * T * d * h / ms / 1e9
        ms = t_ms(lambda: K.grouped_gemm(x, w1t, None, gelu=False, out=out))
        res[f"mode{mode}_dense_gemm1_nobias_tflops"] = 2 * T * d * h / ms / 1e9
    K.set_gemm_mode(0)
    ms = t_ms(lambda: K.grouped_gemm(x, w1t, b1, gelu=True, out=out))
    res["dense_gemm1_gelu_ms"] = ms
    res["dense_gemm1_tflops"] = 2 * T * d * h / ms / 1e9
    ms = t_ms(lambda: K.grouped_gemm(x, w1t, None, gelu=False, out=out))
    res["dense_gemm1_nobias_tflops"] = 2 * T * d * h / ms / 1e9
    ms = t_ms(lambda: torch.matmul(x, w1t.t(), out=out))
    res["cublas_gemm1_tflops"] = 2 * T * d * h / ms / 1e9
    hid = torch.randn(T, h, device="cuda").bfloat16()
    w2t = (torch.randn(d, h, device="cuda") / d ** 0.5).bfloat16()
    out2 = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    ms = t_ms(lambda: K.grouped_gemm(hid, w2t, None, out=out2))
    res["dense_gemm2_tflops"] = 2 * T * d * h / ms / 1e9
    ms = t_ms(lambda: torch.matmul(hid, w2t.t(), out=out2))
    res["cublas_gemm2_tflops"] = 2 * T * d * h / ms / 1e9
    # grouped, 8 experts x 4096 rows (cf=2 capacity), ~2048 rows each filled
    C = 4096
    a = torch.randn(N, C, d, device="cuda").bfloat16()
    w1e = (torch.randn(N, h, d, device="cuda") / d ** 0.5).bfloat16()
    b1e = torch.zeros(N, h, device="cuda")
    rows = torch.full((N,), T // N, device="cuda", dtype=torch.int32)
    o = torch.empty(N, C, h, device="cuda", dtype=torch.bfloat16)
    ms = t_ms(lambda: K.grouped_gemm(a, w1e, b1e, group_rows=rows, rows_clip=C, gelu=True, out=o))
    res["grouped_gemm1_tflops"] = 2 * T * d * h / ms / 1e9
    # gate / dispatch / combine
    wg = torch.randn(N, d, device="cuda") / d ** 0.5
    ms = t_ms(lambda: K.gate_topk(x, wg, 1, C))
    res["gate_ms"] = ms
    res["gate_GBps"] = (T * d * 2 + T * N * 4) / ms / 1e6
    dec = K.gate_topk(x, wg, 1, C)
    buf = torch.empty(N, C, d, device="cuda", dtype=torch.bfloat16)
    ms = t_ms(lambda: K.dispatch(x, dec.indices, dec.slots, N, C, out=buf))
    res["dispatch_GBps"] = 2 * T * d * 2 / ms / 1e6
    se = torch.randn(T, d, device="cuda").bfloat16()
    ms = t_ms(lambda: K.combine(buf, dec.indices, dec.slots, dec.weights, C, se_out=se, residual=x))
    res["combine_GBps"] = 4 * T * d * 2 / ms / 1e6
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
