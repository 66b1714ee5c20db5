"""Tile / epilogue sweep of the configs[1] FFN2 data gradient with the
gelu'-multiply epilogue (dz = (dy W2) * gelu'(z): 18432 x 384 -> 1536,
EPI_MUL_AUX, W read MN-major), at all SMs and at half (the concurrent
backward), vs the plain dgrad; us per call, 20 back-to-back launches,
interleaved rounds, medians."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_05019_b200 import kernels as K, _lib as L
M, Kd, N = 18432, 384, 1536
dy = torch.randn(1, M, Kd, device="cuda").bfloat16()
w2 = (torch.randn(1, Kd, N, device="cuda") / 20).bfloat16()
z = torch.randn(1, M, N, device="cuda").bfloat16()
out = torch.empty(1, M, N, device="cuda").bfloat16()
half = torch.cuda.get_device_properties(0).multi_processor_count // 2
arms = {}
for sms in (0, half):
    for mode in (1, 2):
        for bn in (128, 256):
            for epi in (8, 16):
                def f(mode=mode, bn=bn, epi=epi, sms=sms):
                    K.set_gemm_mode(mode); K.set_gemm_tile_n(bn); K.set_gemm_epilogue_warps(epi)
                    with K.gemm_sm_budget(sms):
                        K.grouped_gemm_ex(dy, w2, L.W_KN, N, aux_in=z, epilogue=L.EPI_MUL_AUX, out=out)
                arms[f"sms{sms or 'all'} m{mode} bn{bn} e{epi}"] = f
for f in arms.values():
    f()
torch.cuda.synchronize()
res = {k: [] for k in arms}
for r in range(4):
    for k, f in arms.items():
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        res[k].append(e0.elapsed_time(e1) / 20 * 1e3)
K.set_gemm_mode(0); K.set_gemm_tile_n(0); K.set_gemm_epilogue_warps(0)
for k, v in sorted(res.items(), key=lambda kv: statistics.median(kv[1])):
    print(f"{k:24s} {statistics.median(v):7.1f} us")
