"""One launch each of the HBM-bound kernels at the configs[2] shape, for
`ncu --set full` (gate: tensor-core and FMA logit paths; dispatch; combine)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2404_05019_b200 import _lib
from paper_2404_05019_b200 import kernels as K

T, d, N, cf = 16384, 2048, 8, 2.0
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(T, d, device="cuda", generator=g).bfloat16()
w = torch.randn(N, d, device="cuda", generator=g) / d ** 0.5
quota = K.expert_quota(cf, T, 1, N)
flag = ctypes.c_int.in_dll(_lib.lib(), "scmoe_gate_force_fma")
flag.value = 0
dec = K.gate_topk(x, w, 1, quota)
flag.value = 1
K.gate_topk(x, w, 1, quota)
flag.value = 0
buf = K.dispatch(x, dec.indices, dec.slots, N, quota)
se = torch.randn(T, d, device="cuda", generator=g).bfloat16()
res = torch.randn(T, d, device="cuda", generator=g).bfloat16()
K.combine(buf, dec.indices, dec.slots, dec.weights, quota, se_out=se, residual=res)
torch.cuda.synchronize()
print("ok")
