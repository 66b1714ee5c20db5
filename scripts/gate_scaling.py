"""Gate kernel time vs token count (d 2048, N 8, top-1, presplit weights,
cold L2): fits time = fixed + bytes / rate to split launch/tail overhead from
streaming.  Device time per launch from CUPTI."""
import os, sys
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2404_05019_b200 import kernels as K
d, N = 2048, 8
w = torch.randn(N, d, device="cuda") / d ** 0.5
ws = K.gate_split_weights(w)
flush = torch.ones(128 * 1024 * 1024, device="cuda")
res = []
for T in (2048, 4096, 8192, 16384, 32768, 65536):
    x = torch.randn(T, d, device="cuda").bfloat16()
    quota = K.expert_quota(2.0, T, 1, N)
    for _ in range(3):
        K.gate_topk(x, w, 1, quota, w_split=ws)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(8):
            flush.sum()
            K.gate_topk(x, w, 1, quota, w_split=ws)
        torch.cuda.synchronize()
    ts = [e.device_time_total for e in prof.events()
          if e.device_type == torch.autograd.DeviceType.CUDA and "gate_topk_tc" in e.name]
    us = sorted(ts)[len(ts) // 2]
    res.append((T, us))
    print(f"T {T:6d}  {us:7.1f} us  {T * d * 2 / us / 1e3:7.0f} GB/s")
import numpy as np
A = np.array([[1, t * d * 2] for t, _ in res], dtype=float)
y = np.array([u for _, u in res])
c, *_ = np.linalg.lstsq(A, y, rcond=None)
print(f"fit: fixed {c[0]:.1f} us, streaming {1 / c[1] / 1e3:.0f} GB/s")
