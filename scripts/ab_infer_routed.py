import os, random, statistics, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2404_05019_b200 as P
from paper_2404_05019_b200.runtime import CapturedStep
T, d, h, N = 16384, 2048, 8192, 8
blk = P.ScMoEBlockPair(d, h, N, variant="scmoe", shortcut_pos="pos2", n_heads=32, seq_len=2048,
                       causal=True, capacity_factor=2.0, dtype=torch.bfloat16,
                       generator=torch.Generator(device="cuda").manual_seed(1))
t2 = P.ScMoEBlockPair(d, h, N, variant="standard", k_routed=2, n_heads=32, seq_len=2048,
                      causal=True, capacity_factor=2.0, dtype=torch.bfloat16,
                      generator=torch.Generator(device="cuda").manual_seed(2))
x = torch.randn(T, d, device="cuda").bfloat16()
graphs = {}
with torch.no_grad():
    import paper_2404_05019_b200.block as B
    for val in (False, True, "decode"):
        blk.routed_stream_infer = val
        graphs[val] = CapturedStep(lambda xx: blk(xx)[0], [x])
    blk.routed_stream_infer = True
    B.SHARED_SPLIT_JOIN = False
    graphs["no-split"] = CapturedStep(lambda xx: blk(xx)[0], [x])
    B.SHARED_SPLIT_JOIN = True
    graphs["top2"] = CapturedStep(lambda xx: t2(xx)[0], [x])
    ref = graphs[False].replay().clone()
    for k in (True, "decode", "no-split"):
        print(k, "identical:", torch.equal(ref, graphs[k].replay().clone()))
    res = {k: [] for k in graphs}
    rng = random.Random(0)
    for r in range(int(os.environ.get("ROUNDS", "12"))):
        items = list(graphs.items())
        rng.shuffle(items)                 # power-cap drift hits every arm alike
        for val, g in items:
            for _ in range(2): g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10): g.replay()
            e1.record(); torch.cuda.synchronize()
            res[val].append(e0.elapsed_time(e1) / 10)
for val, v in res.items():
    print(f"routed_stream_infer={val}: median {statistics.median(v):.3f} ms")
print("top-2 / ScMoE: serial %.3f  side %.3f" % (statistics.median(res["top2"]) / statistics.median(res[False]),
                                               statistics.median(res["top2"]) / statistics.median(res[True])))
