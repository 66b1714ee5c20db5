"""A/B: configs[1] training step with the packed flash-attn path vs cuDNN SDPA
(CUDA-graph replays, interleaved rounds)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P
from paper_2404_05019_b200 import block as B
from paper_2404_05019_b200.runtime import CapturedStep
T, d, h = 18432, 384, 1536
x = torch.randn(T, d, device="cuda").bfloat16()
res = {}
graphs = {}
MODES = ("cudnn_packed", "flash_packed", "autograd")
for packed in MODES:
    B.ATTN_TRAIN = packed
    blk = P.ScMoEBlockPair(d, h, 1, variant="scmoe", shortcut_pos="pos2", n_heads=12, seq_len=144,
                           capacity_factor=1.25, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
    graphs[packed] = CapturedStep(lambda xx, blk=blk: blk.train_step(xx, lr=1e-4), [x], warmup=3)
for r in range(6):
    for packed in MODES:
        B.ATTN_TRAIN = packed
        g = graphs[packed]
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            g.replay()
        b.record(); torch.cuda.synchronize()
        res.setdefault(packed, []).append(a.elapsed_time(b) / 10)
for k, v in res.items():
    print(f"{k:14s} {statistics.median(v):.3f} ms/step", [round(t, 3) for t in v])
