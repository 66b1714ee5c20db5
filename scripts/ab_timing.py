"""A/B device timing of the configs[2] ScMoE and top-2 block pairs, eager and
CUDA-graph replay, interleaved rounds (guards against clock drift)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P
from paper_2404_05019_b200.runtime import CapturedStep

T, d, h, N = 16384, 2048, 8192, 8
kw = dict(n_heads=32, seq_len=2048, causal=True, capacity_factor=2.0, dtype=torch.bfloat16)
sc = P.ScMoEBlockPair(d, h, N, variant="scmoe", shortcut_pos="pos2",
                      generator=torch.Generator(device="cuda").manual_seed(1), **kw)
t2 = P.ScMoEBlockPair(d, h, N, variant="standard", k_routed=2,
                      generator=torch.Generator(device="cuda").manual_seed(1), **kw)
x = torch.randn(T, d, device="cuda").bfloat16()
with torch.no_grad():
    g_sc = CapturedStep(lambda xx: sc(xx)[0], [x])
    g_t2 = CapturedStep(lambda xx: t2(xx)[0], [x])
    cases = {"sc_eager": lambda: sc(x), "t2_eager": lambda: t2(x),
             "sc_graph": g_sc.replay, "t2_graph": g_t2.replay,
             "sc_layer": lambda: sc.moe(x, x), "t2_layer": lambda: t2.moe(x)}
    res = {k: [] for k in cases}
    for rnd in range(4):
        for k, f in cases.items():
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(20):
                f()
            e.record()
            torch.cuda.synchronize()
            res[k].append(s.elapsed_time(e) / 20)
for k, v in res.items():
    print(f"{k:10s} median {statistics.median(v):.3f} ms  all {[round(a, 3) for a in v]}")
