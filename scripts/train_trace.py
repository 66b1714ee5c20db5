"""Per-launch device times of one configs[1] training step, in issue order
(torch.profiler / CUPTI, warm, eager): which launch of the step is slow.

    python scripts/train_trace.py [n_experts] [variant]"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2404_05019_b200 as P

n_exp = int(sys.argv[1]) if len(sys.argv) > 1 else 1
variant = sys.argv[2] if len(sys.argv) > 2 else "scmoe"
T, d, h = 18432, 384, 1536
blk = P.ScMoEBlockPair(d, h, n_exp, variant=variant, k_routed=1 if variant == "scmoe" else 2,
                       shortcut_pos="pos2" if variant == "scmoe" else None, n_heads=12,
                       seq_len=144, capacity_factor=1.25, dtype=torch.bfloat16,
                       generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
x = torch.randn(T, d, device="cuda").bfloat16()
for _ in range(3):
    blk.train_step(x, lr=1e-4)
torch.cuda.synchronize()
graph = os.environ.get("GRAPH", "0") == "1"      # GRAPH=1: one CUDA-graph replay (as the bench)
if graph:
    from paper_2404_05019_b200.runtime import CapturedStep
    g = CapturedStep(lambda xx: blk.train_step(xx, lr=1e-4), [x], warmup=3)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    if graph:
        g.replay()
    else:
        blk.train_step(x, lr=1e-4)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
tot = 0.0
print(f"# {variant} n_experts={n_exp}: {len(evs)} launches")
print("| # | start us | dur us | gap after prev end | kernel |\n|---:|---:|---:|---:|---|")
for i, e in enumerate(evs):
    dur = e.time_range.end - e.time_range.start
    tot += dur
    gap = e.time_range.start - (evs[i - 1].time_range.end if i else e.time_range.start)
    print(f"| {i} | {e.time_range.start - t0:.1f} | {dur:.1f} | {gap:.1f} | `{e.name[:90]}` |")
print(f"# kernel time {tot:.1f} us, span {evs[-1].time_range.end - t0:.1f} us")
