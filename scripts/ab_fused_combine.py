"""A/B: configs[2] ScMoE block pair with the combine fused into the shared
expert's GEMM2 epilogue vs the separate combine kernel (CUDA-graph replays,
interleaved rounds, medians)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P
from paper_2404_05019_b200 import layers as L
from paper_2404_05019_b200.runtime import CapturedStep
T, d, h, N = 16384, 2048, 8192, 8
blk = P.ScMoEBlockPair(d, h, N, variant="scmoe", shortcut_pos="pos2", n_heads=32, seq_len=2048,
                       causal=True, capacity_factor=2.0, dtype=torch.bfloat16,
                       generator=torch.Generator(device="cuda").manual_seed(1))
x = torch.randn(T, d, device="cuda").bfloat16()
graphs = {}
with torch.no_grad():
    for fused in (True, False):
        L.FUSED_COMBINE = fused
        graphs[fused] = CapturedStep(lambda xx: blk(xx)[0], [x])
    res = {}
    for r in range(8):
        for fused in (True, False):
            g = graphs[fused]
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                g.replay()
            b.record(); torch.cuda.synchronize()
            res.setdefault(fused, []).append(a.elapsed_time(b) / 10)
    o1 = graphs[True].replay(); o2 = graphs[False].replay()
    torch.cuda.synchronize()
for k, v in res.items():
    print("fused  " if k else "unfused", f"{statistics.median(v):.4f} ms/step", [round(t, 3) for t in v])
