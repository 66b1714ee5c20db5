"""Gate launches at the configs[2] shape (T 16384, d 2048, N 8), cold L2
(read-only 512 MB flush before each call), per-kernel device time from CUPTI."""
import os, sys
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2404_05019_b200 as P
T, d, N = 16384, 2048, 8
moe = P.ScMoELayer(d, 8192, N, capacity_factor=2.0, dtype=torch.bfloat16,
                   generator=torch.Generator(device="cuda").manual_seed(1))
x = torch.randn(T, d, device="cuda").bfloat16()
flush = torch.ones(128 * 1024 * 1024, device="cuda")
with torch.no_grad():
    for _ in range(3):
        moe.route(x)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            flush.sum()
            moe.route(x)
        torch.cuda.synchronize()
agg = defaultdict(list)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        agg[e.name].append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):4d} {sum(v) / len(v):8.1f} us  {k[:110]}")
