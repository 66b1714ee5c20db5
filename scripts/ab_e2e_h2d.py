"""e2e through HostStreamRunner with the input copies on one stream vs two
concurrent halves (configs[2] block pair, CUDA graphs, 20 steps, interleaved
rounds, medians).  Needs a runner with an `h2d_b` stream (the two-stream
variant was measured 4.235 vs 4.191 ms/step — slower — and not kept, so this
script documents the experiment)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P
from paper_2404_05019_b200.runtime import CapturedStep, HostStreamRunner
T, d = 16384, 2048
blk = P.ScMoEBlockPair(d, 8192, 8, variant="scmoe", shortcut_pos="pos2", n_heads=32, seq_len=2048,
                       causal=True, capacity_factor=2.0, dtype=torch.bfloat16,
                       generator=torch.Generator(device="cuda").manual_seed(1))
x = torch.randn(T, d, device="cuda").bfloat16()
h = torch.empty(T, d, dtype=torch.bfloat16, pin_memory=True)
h.copy_(x.cpu())
outs = [torch.empty(T, d, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
steps = 20
with torch.no_grad():
    runners = {}
    for name in ("one_stream", "two_streams"):
        r = HostStreamRunner([CapturedStep(lambda xx: blk(xx)[0], [x]),
                              CapturedStep(lambda xx: blk(xx)[0], [x])])
        if name == "one_stream":
            r.h2d_b = r.h2d
        runners[name] = r
        r.run([h] * 3, [outs[i % 2] for i in range(3)])
    res = {k: [] for k in runners}
    for rnd in range(6):
        for name, r in runners.items():
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r.run([h] * steps, [outs[i % 2] for i in range(steps)])
            e1.record()
            torch.cuda.synchronize()
            res[name].append(e0.elapsed_time(e1) / steps)
for k, v in res.items():
    print(f"{k:12s} e2e median {statistics.median(v):.3f} ms/step")
