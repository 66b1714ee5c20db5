"""ncu / timing target: configs[1] training step (SwinV2-MoE-S stage-3 ScMoE
block pair, T=18432, d=384, h=1536, 1 expert, cf 1.25, bf16)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
T, d, h = 18432, 384, 1536
blk = P.ScMoEBlockPair(d, h, 1, variant="scmoe", shortcut_pos="pos2", n_heads=12, seq_len=144,
                       capacity_factor=1.25, dtype=torch.bfloat16,
                       generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
x = torch.randn(T, d, device="cuda").bfloat16()
for _ in range(3):
    blk.train_step(x, lr=1e-4)
torch.cuda.synchronize()
t0 = time.perf_counter()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(steps):
    blk.train_step(x, lr=1e-4)
e.record()
torch.cuda.synchronize()
print(f"device ms/step {s.elapsed_time(e)/steps:.3f}  host ms/step {(time.perf_counter()-t0)*1e3/steps:.3f}")
