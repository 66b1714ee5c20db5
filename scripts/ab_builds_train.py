"""A/B two builds of libscmoe.so on the configs[1] training step (CUDA-graph
replays), one subprocess per measurement, builds interleaved:

    python scripts/ab_builds_train.py libA.so libB.so [rounds] [n_experts]
"""
import json, os, statistics, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_2404_05019_b200 as P
from paper_2404_05019_b200.runtime import CapturedStep
n = int(os.environ["NEXP"])
T, d, h = 18432, 384, 1536
blk = P.ScMoEBlockPair(d, h, n, variant="scmoe", shortcut_pos="pos2", n_heads=12, seq_len=144,
                       capacity_factor=1.25, dtype=torch.bfloat16,
                       generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
x = torch.randn(T, d, device="cuda").bfloat16()
g = CapturedStep(lambda xx: blk.train_step(xx, lr=1e-4), [x], warmup=3)
for _ in range(5): g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(30): g.replay()
b.record(); torch.cuda.synchronize()
print(json.dumps({"us": a.elapsed_time(b) / 30 * 1e3}))
'''
libs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 4
nexp = sys.argv[4] if len(sys.argv) > 4 else "1"
res = {l: [] for l in libs}
for r in range(rounds):
    for lib in libs:
        env = dict(os.environ, SCMOE_LIB=os.path.abspath(lib), ROOT=ROOT, NEXP=nexp)
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if not line:
            print(out.stderr[-2000:]); sys.exit(1)
        res[lib].append(json.loads(line[-1])["us"])
for lib, v in res.items():
    print(f"{os.path.basename(lib):24s} median {statistics.median(v):.1f} us  {[round(t) for t in v]}")
