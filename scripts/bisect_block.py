"""Which op of the d=128 block pair changes with the GEMM tile width?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P
from paper_2404_05019_b200 import kernels as K
T, d, h, N = 256, 128, 256, 4
blk = P.ScMoEBlockPair(d, h, N, variant="scmoe", shortcut_pos="pos2", dtype=torch.bfloat16,
                       generator=torch.Generator(device="cuda").manual_seed(1))
x = torch.randn(T, d, device="cuda").bfloat16()
res = {}
for bn in (256, 0):
    K.set_gemm_tile_n(bn)
    with torch.no_grad():
        out, dec, aux, taps = blk(x, return_taps=True)
    torch.cuda.synchronize()
    res[bn] = dict(taps, out=out)
K.set_gemm_tile_n(0)
for k in res[0]:
    a, b = res[256][k].float(), res[0][k].float()
    print(k, float((a - b).abs().max()), float(a.abs().max()))
a = torch.randn(256, 128, device="cuda").bfloat16()
for n in (128, 384):
    w = torch.randn(n, 128, device="cuda").bfloat16()
    for mode in (1, 2):
        K.set_gemm_mode(mode)
        outs = {}
        for bn in (256, 192):
            K.set_gemm_tile_n(bn)
            outs[bn] = K.grouped_gemm(a, w, None)
        torch.cuda.synchronize()
        print("gemm n", n, "mode", mode, float((outs[256].float() - outs[192].float()).abs().max()))
K.set_gemm_mode(0); K.set_gemm_tile_n(0)
