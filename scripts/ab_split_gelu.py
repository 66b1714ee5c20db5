"""A/B of the training FFN's GELU placement (training.SPLIT_GELU): the
configs[1] training step as a CUDA graph, interleaved rounds, medians.

    python scripts/ab_split_gelu.py [n_experts]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P
from paper_2404_05019_b200 import training as TR
from paper_2404_05019_b200.runtime import CapturedStep

n_exp = int(sys.argv[1]) if len(sys.argv) > 1 else 1
T, d, h = 18432, 384, 1536
x = torch.randn(T, d, device="cuda").bfloat16()
graphs = {}
for split in (False, True):
    TR.SPLIT_GELU = split
    blk = P.ScMoEBlockPair(d, h, n_exp, variant="scmoe", shortcut_pos="pos2", n_heads=12,
                           seq_len=144, capacity_factor=1.25, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
    graphs[split] = (blk, CapturedStep(lambda xx, b=blk: b.train_step(xx, lr=1e-4), [x], warmup=3))
res = {False: [], True: []}
for r in range(6):
    for split in (False, True):
        g = graphs[split][1]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[split].append(e0.elapsed_time(e1) / 10)
for split in (False, True):
    print(f"SPLIT_GELU={split}: {statistics.median(res[split]):.3f} ms/step  {res[split]}")
