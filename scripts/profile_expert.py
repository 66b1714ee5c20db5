"""ncu target: the routed-expert FFN of the configs[2] ScMoE layer
(T=16384, d=2048, h=8192, N=8, cf=2): route + dispatch once, then the two
grouped-GEMM launches (GEMM1 bias+GELU, GEMM2 bias) `--iters` times.

  ncu --set full -k regex:grouped_gemm -s 2 -c 2 -o prof python scripts/profile_expert.py
captures iteration 2's GEMM1 and GEMM2.
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--shape", default="cfg2", choices=["cfg2", "cfg3"])   # cfg3: T 8192, d 4096, h 16384, N 16
ap.add_argument("--flags", type=int, default=0)                       # scmoe_set_gemm_flags
a = ap.parse_args()
T, d, h, N = (16384, 2048, 8192, 8) if a.shape == "cfg2" else (8192, 4096, 16384, 16)
gen = torch.Generator(device="cuda").manual_seed(3)
layer = P.ScMoELayer(d, h, N, capacity_factor=2.0, dtype=torch.bfloat16, generator=gen)
x = torch.randn(T, d, device="cuda", generator=gen).bfloat16()
from paper_2404_05019_b200 import kernels as K
K.set_gemm_mode(a.mode)
K.set_gemm_flags(a.flags)
with torch.no_grad():
    dec = layer.route(x)
    buf = K.dispatch(x, dec.indices, dec.slots, N, dec.capacity)
    for _ in range(a.iters):
        y = layer.experts(buf, dec.counts, dec.capacity)
torch.cuda.synchronize()
print("kept rows", int(dec.kept_counts().sum()), "capacity", dec.capacity)
