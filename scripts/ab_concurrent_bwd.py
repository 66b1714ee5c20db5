"""A/B of training.CONCURRENT_BWD (data- and weight-gradient GEMMs of a layer
on two streams, half the SMs each) on the configs[1] training step, CUDA-graph
replays, interleaved rounds, medians."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P
from paper_2404_05019_b200 import training as TR
from paper_2404_05019_b200.runtime import CapturedStep
n_exp = int(sys.argv[1]) if len(sys.argv) > 1 else 1
T, d, h = 18432, 384, 1536
x = torch.randn(T, d, device="cuda").bfloat16()
graphs = {}
for conc in (False, True):
    TR.CONCURRENT_BWD = conc
    blk = P.ScMoEBlockPair(d, h, n_exp, variant="scmoe", shortcut_pos="pos2", n_heads=12, seq_len=144,
                           capacity_factor=1.25, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
    graphs[conc] = CapturedStep(lambda xx, b=blk: b.train_step(xx, lr=1e-4), [x], warmup=3)
res = {False: [], True: []}
for r in range(6):
    for conc, g in graphs.items():
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[conc].append(e0.elapsed_time(e1) / 20)
for conc, v in res.items():
    print(f"concurrent={conc}: median {statistics.median(v) * 1e3:.1f} us  {[round(t * 1e3) for t in v]}")
