import os, sys
sys.path.insert(0, "/root/repo")
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2404_05019_b200 as P
T, d, h = 18432, 384, 1536
blk = P.ScMoEBlockPair(d, h, 1, variant="scmoe", shortcut_pos="pos2", n_heads=12, seq_len=144,
                       capacity_factor=1.25, dtype=torch.bfloat16,
                       generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
x = torch.randn(T, d, device="cuda").bfloat16()
for _ in range(3): blk.train_step(x, lr=1e-4)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=True, record_shapes=True) as prof:
    blk.train_step(x, lr=1e-4)
    torch.cuda.synchronize()
for e in prof.events():
    if e.name in ("aten::copy_", "aten::add", "aten::add_", "aten::contiguous", "aten::clone", "aten::to", "aten::_to_copy"):
        st = [s for s in (e.stack or []) if "paper_2404" in s or "site-packages/torch/autograd" in s][:3]
        print(e.name, e.input_shapes[:2] if e.input_shapes else "", st)
