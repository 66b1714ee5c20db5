"""ncu target: one eager configs[1] training step (T 18432, d 384, h 1536,
one expert); capture the step's GEMM launches with

  ncu --set full -k regex:gemm_kernel -s 30 -c 12 python scripts/profile_train_gemms.py

(the first step warms up; -s skips its launches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P
T, d, h = 18432, 384, 1536
blk = P.ScMoEBlockPair(d, h, 1, variant="scmoe", shortcut_pos="pos2", n_heads=12, seq_len=144,
                       capacity_factor=1.25, dtype=torch.bfloat16,
                       generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
x = torch.randn(T, d, device="cuda").bfloat16()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    blk.train_step(x, lr=1e-4)
torch.cuda.synchronize()
