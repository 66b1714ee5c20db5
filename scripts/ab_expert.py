"""A/B of builds of libscmoe.so on the routed-expert FFN of the configs[2]
ScMoE layer (T=16384, d=2048, h=8192, N=8, cf=2): GEMM1 (bias+GELU) and
GEMM2 (bias) CUPTI durations, medians over iterations, builds interleaved in
subprocesses on the same box.  Also the dense configs[2] FFN (mlp_prev shape:
one group of 16384 rows) as a control.

    python scripts/ab_expert.py libA.so libB.so [rounds]
"""
import json, os, statistics, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_2404_05019_b200 as P
from paper_2404_05019_b200 import kernels as K
from torch.profiler import profile, ProfilerActivity
T, d, h, N = 16384, 2048, 8192, 8
gen = torch.Generator(device="cuda").manual_seed(3)
layer = P.ScMoELayer(d, h, N, capacity_factor=2.0, dtype=torch.bfloat16, generator=gen)
x = torch.randn(T, d, device="cuda", generator=gen).bfloat16()
w1 = (torch.randn(h, d, device="cuda", generator=gen) * 0.02).bfloat16()
w2 = (torch.randn(d, h, device="cuda", generator=gen) * 0.02).bfloat16()
b1 = torch.zeros(h, device="cuda"); b2 = torch.zeros(d, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
K.set_gemm_epilogue_warps(int(os.environ.get("SCMOE_EPI", "0")))
with torch.no_grad():
    dec = layer.route(x)
    buf = K.dispatch(x, dec.indices, dec.slots, N, dec.capacity)
    def routed():
        layer.experts(buf, dec.counts, dec.capacity)
    def dense():
        hh = K.grouped_gemm(x, w1, b1, gelu=True)
        K.grouped_gemm(hh, w2, b2)
    for f in (routed, dense):
        for _ in range(3): f()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(int(os.environ.get("ITERS", "8"))):
            for f in (routed, dense):
                flush.zero_()
                f()
        torch.cuda.synchronize()
ks = [e for e in prof.events() if e.device_type.name == "CUDA" and "gemm_kernel" in e.name]
# order per iteration: routed g1, routed g2, dense g1, dense g2
names = ["routed_g1", "routed_g2", "dense_g1", "dense_g2"]
res = {n: [] for n in names}
for i, e in enumerate(ks):
    res[names[i % 4]].append(e.device_time if hasattr(e, "device_time") else e.cuda_time)
print(json.dumps({k: sorted(v)[len(v) // 2] for k, v in res.items()}))
'''
libs = sys.argv[1:3]
# "lib.so@16": the same build with 16 epilogue warps forced (SCMOE_EPI)
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
res = {l: [] for l in libs}
for r in range(rounds):
    for lib in libs:
        path, _, epi = lib.partition("@")
        env = dict(os.environ, SCMOE_LIB=os.path.abspath(path), ROOT=ROOT, SCMOE_EPI=epi or "0")
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if not line:
            print(out.stderr[-3000:]); sys.exit(1)
        res[lib].append(json.loads(line[-1]))
for lib, v in res.items():
    keys = v[0].keys()
    print(f"{os.path.basename(lib):24s} " + "  ".join(
        f"{k} {statistics.median([x[k] for x in v]):.1f}us" for k in keys))
