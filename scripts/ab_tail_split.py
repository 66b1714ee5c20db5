"""Routed-expert FFN at configs[2] (T 16384, d 2048, h 8192, N 8, cf 2):
tail split on vs off, interleaved rounds, median ms of the two GEMMs."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_05019_b200 as P
from paper_2404_05019_b200 import kernels as K
T, d, h, N = 16384, 2048, 8192, 8
layer = P.ScMoELayer(d, h, N, capacity_factor=2.0, dtype=torch.bfloat16,
                     generator=torch.Generator(device="cuda").manual_seed(3))
x = torch.randn(T, d, device="cuda").bfloat16()
with torch.no_grad():
    dec = layer.route(x)
    buf = K.dispatch(x, dec.indices, dec.slots, N, dec.capacity)
    print("rows per expert", dec.kept_counts().tolist())
    res = {}
    for _ in range(2):
        for on in (True, False):
            K.set_gemm_tail_split(on)
            layer.experts(buf, dec.counts, dec.capacity)
    for r in range(6):
        for on in (True, False):
            K.set_gemm_tail_split(on)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                layer.experts(buf, dec.counts, dec.capacity)
            e1.record(); torch.cuda.synchronize()
            res.setdefault(on, []).append(e0.elapsed_time(e1) / 10)
    K.set_gemm_tail_split(True)
for on, v in res.items():
    print(f"tail split {on}: {statistics.median(v):.3f} ms")
