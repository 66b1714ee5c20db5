"""A/B of GEMM launch flags (scmoe_set_gemm_flags; bit 3 = programmatic
dependent launch off) on the configs[1] training step and the configs[2]
inference block pair: one CUDA graph per setting, captured under that
setting, interleaved rounds, medians.

    python scripts/ab_flags.py FLAGS_A FLAGS_B"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2404_05019_b200 as P
from paper_2404_05019_b200 import _lib as L
from paper_2404_05019_b200.runtime import CapturedStep

fa, fb = int(sys.argv[1]), int(sys.argv[2])
which = sys.argv[3] if len(sys.argv) > 3 else "train,infer"
xt = torch.randn(18432, 384, device="cuda").bfloat16()
xi = torch.randn(16384, 2048, device="cuda").bfloat16()
arms = {}
for f in (fa, fb):
    L.lib().scmoe_set_gemm_flags(f)
    tr = P.ScMoEBlockPair(384, 1536, 1, variant="scmoe", shortcut_pos="pos2", n_heads=12,
                          seq_len=144, capacity_factor=1.25, dtype=torch.bfloat16,
                          generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
    if "train" in which:
        arms[("train", f)] = CapturedStep(lambda xx, b=tr: b.train_step(xx, lr=1e-4), [xt])
    if "infer" not in which:
        continue
    inf = P.ScMoEBlockPair(2048, 8192, 8, variant="scmoe", shortcut_pos="pos2", n_heads=32,
                           seq_len=2048, causal=True, capacity_factor=2.0, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(1))
    with torch.no_grad():
        arms[("infer", f)] = CapturedStep(lambda xx, b=inf: b(xx)[0], [xi])
L.lib().scmoe_set_gemm_flags(0)
res = {k: [] for k in arms}
for _ in range(6):
    for k, g in arms.items():
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[k].append(e0.elapsed_time(e1) / 10)
for k, v in res.items():
    print(f"{k[0]:6s} flags={k[1]:2d}: {statistics.median(v):.4f} ms  {[round(t, 3) for t in v]}")
