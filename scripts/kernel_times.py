"""Warm per-kernel device time (torch.profiler / CUPTI) of the bench steps.

    python scripts/kernel_times.py train|infer [steps]

Prints a table: kernel, launches per step, us per step, share — the warm
counterpart of the ncu launch list (which is cold-cache and serialised)."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2404_05019_b200 as P

mode = sys.argv[1] if len(sys.argv) > 1 else "train"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if mode == "train":
    T, d, h = 18432, 384, 1536
    blk = P.ScMoEBlockPair(d, h, 1, variant="scmoe", shortcut_pos="pos2", n_heads=12, seq_len=144,
                           capacity_factor=1.25, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
    x = torch.randn(T, d, device="cuda").bfloat16()
    fn = lambda: blk.train_step(x, lr=1e-4)
else:
    T, d, h = 16384, 2048, 8192
    blk = P.ScMoEBlockPair(d, h, 8, variant="scmoe", shortcut_pos="pos2", n_heads=32, seq_len=2048,
                           causal=True, capacity_factor=2.0, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(1))
    x = torch.randn(T, d, device="cuda").bfloat16()

    def fn():
        with torch.no_grad():
            blk(x)
for _ in range(3):
    fn()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        fn()
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        a = agg[ev.name]
        a[0] += 1
        a[1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v[1] for v in agg.values())
print(f"# {mode}: {tot / steps:.1f} us of kernel time per step ({steps} steps)")
print("| launches/step | us/step | share | kernel |\n|---:|---:|---:|---|")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"| {n / steps:.1f} | {t / steps:.1f} | {100 * t / tot:.1f}% | `{k[:100]}` |")
