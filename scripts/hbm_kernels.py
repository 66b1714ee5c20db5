"""Device time and achieved HBM bandwidth of the HBM-bound kernels (K1 gate,
K2 dispatch, K5 combine) at the configs[2] shape, L2 flushed before every
launch, CUDA events on the launching stream.

    python scripts/hbm_kernels.py [reps]

Algorithmic bytes per launch:
  gate     T*d*2 (x) + T*N*4 (logits)
  dispatch (rows read + kept rows written)*d*2 (a token row is read once)
  combine  (k+3)*T*d*2 (expert rows + SE + residual, output write)
"""
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2404_05019_b200 import _lib
from paper_2404_05019_b200 import kernels as K

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
T, d, N, cf = 16384, 2048, 8, 2.0
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(T, d, device="cuda", generator=g).bfloat16()
w = torch.randn(N, d, device="cuda", generator=g) / d ** 0.5
flush = torch.ones(128 * 1024 * 1024, dtype=torch.float32, device="cuda")   # read-only L2 flush
st = torch.cuda.current_stream()
peaks = {}
pp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
if os.path.exists(pp):
    peaks = json.load(open(pp))
hbm = peaks.get("hbm_gbs", 6547.2)


def time_us(fn):
    ts = []
    for i in range(reps + 3):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)   # keep the GPU busy while the host enqueues fn
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


res = {}
flag = ctypes.c_int.in_dll(_lib.lib(), "scmoe_gate_force_fma")
for k in (1, 2):
    quota = K.expert_quota(cf, T, k, N)
    for name, f in (("mma", 0), ("fma", 1)):
        flag.value = f
        us = time_us(lambda: K.gate_topk(x, w, k, quota))
        by = T * d * 2 + T * N * 4
        res[f"gate_k{k}_{name}"] = dict(us=us, gbps=by / us / 1e3)
    flag.value = 0
    dec = K.gate_topk(x, w, k, quota)
    kept = int((dec.slots < quota).sum().item())
    buf = K.dispatch(x, dec.indices, dec.slots, N, quota)
    dflag = ctypes.c_int.in_dll(_lib.lib(), "scmoe_dispatch_force_ldst")
    for name, f in (("bulk", 0), ("ldst", 1)):
        dflag.value = f
        us = time_us(lambda: K.dispatch(x, dec.indices, dec.slots, N, quota, out=buf))
        # each token row is read once and written to every kept selection
        rd = int(((dec.slots < quota).any(dim=1)).sum().item())
        res[f"dispatch_k{k}_{name}"] = dict(us=us, gbps=(rd + kept) * d * 2 / us / 1e3)
    dflag.value = 0
    se = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    resid = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    out = torch.empty_like(se)
    us = time_us(lambda: K.combine(buf, dec.indices, dec.slots, dec.weights, quota, se_out=se,
                                   residual=resid, out=out))
    res[f"combine_k{k}"] = dict(us=us, gbps=(k + 3) * T * d * 2 / us / 1e3)
for kk, v in res.items():
    v["frac_hbm"] = v["gbps"] / hbm
    print(f"{kk:16s} {v['us']:8.1f} us  {v['gbps']:7.0f} GB/s  {100 * v['frac_hbm']:5.1f}% of {hbm:.0f}")
print(json.dumps(res))

# the gate inside a CUDA graph (launch gaps as in the bench's graphed step),
# and warm per-kernel times from CUPTI
quota = K.expert_quota(cf, T, 1, N)
K.gate_topk(x, w, 1, quota)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    K.gate_topk(x, w, 1, quota)
    with torch.cuda.graph(g, stream=s):
        K.gate_topk(x, w, 1, quota)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
us = time_us(lambda: g.replay())
print(f"gate_k1 graph     {us:8.1f} us  {(T * d * 2 + T * N * 4) / us / 1e3:7.0f} GB/s")
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        flush.sum()
        g.replay()
    torch.cuda.synchronize()
agg = {}
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA and "gate" in ev.name:
        agg.setdefault(ev.name[:60], []).append(ev.device_time_total)
for kname, v in agg.items():
    print(f"  warm {kname:60s} {statistics.median(v):7.1f} us")
