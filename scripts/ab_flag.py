"""A/B of a boolean module flag on the configs[1] training step (one CUDA
graph per setting, interleaved rounds, medians):

    python scripts/ab_flag.py training.SPLIT_COLSUM [n_experts]
    python scripts/ab_flag.py blk.routed_stream_train [n_experts] [False,gate]   # block attribute
"""
import importlib, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P
from paper_2404_05019_b200.runtime import CapturedStep
modname, flag = sys.argv[1].rsplit(".", 1)
mod = None if modname == "blk" else importlib.import_module("paper_2404_05019_b200." + modname)
n_exp = int(sys.argv[2]) if len(sys.argv) > 2 else 1
T, d, h = 18432, 384, 1536
x = torch.randn(T, d, device="cuda").bfloat16()
graphs = {}
vals = (False, True) if len(sys.argv) <= 3 else tuple(
    {"True": True, "False": False}.get(v, v) for v in sys.argv[3].split(","))
for val in vals:
    if mod is not None:
        setattr(mod, flag, val)
    blk = P.ScMoEBlockPair(d, h, n_exp, variant="scmoe", shortcut_pos="pos2", n_heads=12, seq_len=144,
                           capacity_factor=1.25, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
    if mod is None:
        setattr(blk, flag, val)
    graphs[val] = CapturedStep(lambda xx, b=blk: b.train_step(xx, lr=1e-4), [x], warmup=3)
res = {k: [] for k in graphs}
for r in range(6):
    for val, g in graphs.items():
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[val].append(e0.elapsed_time(e1) / 20 * 1e3)
for val, v in res.items():
    print(f"{flag}={val}: median {statistics.median(v):7.1f} us")
