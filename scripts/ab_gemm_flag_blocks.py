"""A/B of a GEMM experiment flag (scmoe_set_gemm_flags, argv[1], e.g. 32 =
the old n-fastest tile order) on the configs[2] block pair and the configs[3]
every-block block: one CUDA graph per (workload, flag value), shuffled
interleaved rounds, medians; outputs compared bit for bit."""
import os, random, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P
from paper_2404_05019_b200 import kernels as K
from paper_2404_05019_b200.runtime import CapturedStep
flag = int(sys.argv[1]) if len(sys.argv) > 1 else 32
gen = lambda s: torch.Generator(device="cuda").manual_seed(s)
cfg2 = P.ScMoEBlockPair(2048, 8192, 8, variant="scmoe", shortcut_pos="pos2", n_heads=32,
                        seq_len=2048, causal=True, capacity_factor=2.0, dtype=torch.bfloat16,
                        generator=gen(1))
cfg3 = P.ScMoEBlock(4096, 16384, 16, variant="scmoe", shortcut_pos="pos1", n_heads=32,
                    seq_len=2048, causal=True, capacity_factor=2.0, dtype=torch.bfloat16,
                    generator=gen(2))
x2 = torch.randn(16384, 2048, device="cuda", generator=gen(3)).bfloat16()
x3 = torch.randn(8192, 4096, device="cuda", generator=gen(4)).bfloat16()
graphs, outs = {}, {}
with torch.no_grad():
    for name, blk, x in (("cfg2", cfg2, x2), ("cfg3", cfg3, x3)):
        for f in (0, flag):
            K.set_gemm_flags(f)
            graphs[(name, f)] = CapturedStep(lambda xx, b=blk: b(xx)[0], [x])
            outs[(name, f)] = graphs[(name, f)].replay().clone()
        K.set_gemm_flags(0)
        print(name, "identical:", torch.equal(outs[(name, 0)], outs[(name, flag)]))
    res = {k: [] for k in graphs}
    rng = random.Random(0)
    for r in range(int(os.environ.get("ROUNDS", "10"))):
        items = list(graphs.items())
        rng.shuffle(items)
        for k, g in items:
            for _ in range(2):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(8):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) / 8)
for k, v in sorted(res.items()):
    print(f"{k[0]} flags={k[1]:3d}: median {statistics.median(v):.3f} ms")
