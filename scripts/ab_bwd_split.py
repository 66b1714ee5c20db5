"""SM split of the concurrent backward (training.BWD_SIDE_FRAC / BWD_MAIN_FRAC)
on the configs[1] training step: one CUDA graph per setting, interleaved
rounds, medians.   python scripts/ab_bwd_split.py [n_experts]"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P
from paper_2404_05019_b200 import training as TR
from paper_2404_05019_b200.runtime import CapturedStep
n_exp = int(sys.argv[1]) if len(sys.argv) > 1 else 1
T, d, h = 18432, 384, 1536
x = torch.randn(T, d, device="cuda").bfloat16()
settings = {"serial": None, "50/50": (0.5, 0.5), "side50/main-all": (0.5, 0.0),
            "35/65": (0.35, 0.65), "25/75": (0.25, 0.75), "side35/main-all": (0.35, 0.0)}
graphs = {}
for name, st in settings.items():
    TR.CONCURRENT_BWD = st is not None
    if st is not None:
        TR.BWD_SIDE_FRAC, TR.BWD_MAIN_FRAC = st
    blk = P.ScMoEBlockPair(d, h, n_exp, variant="scmoe", shortcut_pos="pos2", n_heads=12, seq_len=144,
                           capacity_factor=1.25, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
    graphs[name] = CapturedStep(lambda xx, b=blk: b.train_step(xx, lr=1e-4), [x], warmup=3)
res = {k: [] for k in graphs}
for r in range(5):
    for name, g in graphs.items():
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / 20 * 1e3)
for name, v in res.items():
    print(f"{name:18s} median {statistics.median(v):7.1f} us")
