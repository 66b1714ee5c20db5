"""A/B two builds of libscmoe.so on the same box: the configs[2] ScMoE block
pair (CUDA-graph replays), one subprocess per measurement, builds interleaved.

    python scripts/ab_builds.py libA.so libB.so [rounds]
"""
import json, os, statistics, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_2404_05019_b200 as P
from paper_2404_05019_b200.runtime import CapturedStep
T, d, h, N = 16384, 2048, 8192, 8
blk = P.ScMoEBlockPair(d, h, N, variant="scmoe", shortcut_pos="pos2", n_heads=32, seq_len=2048,
                       causal=True, capacity_factor=2.0, dtype=torch.bfloat16,
                       generator=torch.Generator(device="cuda").manual_seed(1))
x = torch.randn(T, d, device="cuda").bfloat16()
with torch.no_grad():
    g = CapturedStep(lambda xx: blk(xx)[0], [x])
    for _ in range(5): g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): g.replay()
    b.record(); torch.cuda.synchronize()
print(json.dumps({"ms": a.elapsed_time(b) / 20}))
'''
libs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 4
res = {l: [] for l in libs}
for r in range(rounds):
    for lib in libs:
        env = dict(os.environ, SCMOE_LIB=os.path.abspath(lib), ROOT=ROOT)
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if not line:
            print(out.stderr[-2000:]); sys.exit(1)
        res[lib].append(json.loads(line[-1])["ms"])
for lib, v in res.items():
    print(f"{os.path.basename(lib):24s} median {statistics.median(v):.4f} ms  {[round(t, 3) for t in v]}")
