"""Weight-gradient time vs token count (configs[1] FFN1 shape, 1536 x 384):
fixed cost vs per-token rate, CUPTI device time of the GEMM + split
reduction, medians; back-to-back launches (PDL) as in the step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2404_05019_b200 import kernels as K
M, N = 1536, 384
K.set_gemm_mode(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
res = []
for T in (2304, 4608, 9216, 18432, 36864):
    a = torch.randn(1, T, M, device="cuda").bfloat16()
    b = torch.randn(1, T, N, device="cuda").bfloat16()
    for _ in range(3):
        K.grouped_wgrad(a, b, n_wgroups=1)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            K.grouped_wgrad(a, b, n_wgroups=1)
        torch.cuda.synchronize()
    g = sorted(e.device_time_total for e in prof.events()
               if e.device_type == torch.autograd.DeviceType.CUDA and "gemm_kernel" in e.name)
    r = sorted(e.device_time_total for e in prof.events()
               if e.device_type == torch.autograd.DeviceType.CUDA and "reduce_splits" in e.name)
    gu, ru = g[len(g) // 2], (r[len(r) // 2] if r else 0.0)
    res.append((T, gu, ru))
    print(f"T {T:6d}  gemm {gu:6.1f} us ({2 * T * M * N / gu / 1e6:5.0f} TFLOP/s)  reduce {ru:5.1f} us")
A = np.array([[1, t] for t, _, _ in res], dtype=float)
c, *_ = np.linalg.lstsq(A, np.array([g for _, g, _ in res]), rcond=None)
print(f"fit gemm: {c[0]:.1f} us fixed + {c[1] * 1e3:.2f} us per 1k tokens "
      f"({2 * M * N * 1e3 / (c[1] * 1e3) / 1e6:.0f} TFLOP/s marginal)")
