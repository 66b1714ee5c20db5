"""Device time of the configs[1] training GEMM shapes (M = 18432) under the
epilogue variants: residual or not, 8 / 16 epilogue warps, tile width.
CUDA-graph replays of 20 launches, CUDA events, median of 5.

    python scripts/train_gemm_ab.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2404_05019_b200 import _lib as L
from paper_2404_05019_b200 import kernels as K

M = 18432
torch.manual_seed(0)


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    out = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3 / reps)
    return statistics.median(out)


shapes = [  # name, K, N, layout, bias, residual
    ("o_fwd", 384, 384, L.W_NK, False, True),
    ("o_fwd_nores", 384, 384, L.W_NK, False, False),
    ("ffn2_fwd_res", 1536, 384, L.W_NK, True, True),
    ("ffn2_fwd", 1536, 384, L.W_NK, True, False),
    ("ffn1_dx_res", 1536, 384, L.W_KN, False, True),
    ("ffn1_dx", 1536, 384, L.W_KN, False, False),
    ("qkv_dx_res", 1152, 384, L.W_KN, False, True),
    ("ffn1_fwd", 384, 1536, L.W_NK, True, False),
    ("qkv_fwd", 384, 1152, L.W_NK, False, False),
    ("ffn2_dh", 384, 1536, L.W_KN, False, False),
    ("ffn2_dz_mul", 384, 1536, L.W_KN, False, "mul"),
    ("ffn2_dz_gbwd", 384, 1536, L.W_KN, False, "gbwd"),
    ("ffn1_fwd_gelu_aux", 384, 1536, L.W_NK, True, "gelu_aux"),
]
variants = [(0, 0, 0), (8, 0, 0), (16, 0, 0), (8, 128, 0)]
if len(sys.argv) > 1:     # epi:bn:flags
    variants = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]]
print("| shape | " + " | ".join(f"epi{e}/bn{b}/f{f}" for e, b, f in variants) +
      " | TFLOP/s best |")
print("|---|" + "---:|" * (len(variants) + 1))
for name, Kd, N, lay, bias, res in shapes:
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    w = (torch.randn(N, Kd, device="cuda") / Kd ** 0.5).bfloat16()
    if lay == L.W_KN:
        w = w.t().contiguous()
    b = torch.zeros(N, device="cuda") if bias else None
    r = torch.randn(M, N, device="cuda").bfloat16() if res else None
    kw = dict(bias=b, residual=r)
    if res == "mul":
        kw = dict(aux_in=r, epilogue=L.EPI_MUL_AUX)
    elif res == "gbwd":
        kw = dict(aux_in=r, epilogue=L.EPI_GELU_BWD)
    elif res == "gelu_aux":
        kw = dict(bias=b, aux_out=r, epilogue=L.EPI_BIAS_GELU)
    row = []
    for e, bn, fl in variants:
        K.set_gemm_epilogue_warps(e)
        L.lib().scmoe_set_gemm_tile_n(bn)
        L.lib().scmoe_set_gemm_flags(fl)
        try:
            t = timeit(lambda: K.grouped_gemm_ex(a, w, lay, N, **kw))
        except Exception as ex:  # noqa: BLE001
            t = float("nan")
        row.append(t)
    K.set_gemm_epilogue_warps(0)
    L.lib().scmoe_set_gemm_tile_n(0)
    L.lib().scmoe_set_gemm_flags(0)
    best = min(x for x in row if x == x)
    print(f"| {name} | " + " | ".join(f"{x:.1f}" for x in row) +
          f" | {2 * M * Kd * N / (best * 1e-6) / 1e12:.0f} |")
