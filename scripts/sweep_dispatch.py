import ctypes, statistics, sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2404_05019_b200 import _lib, kernels as K
T, d, N = 16384, 2048, 8
x = torch.randn(T, d, device="cuda").bfloat16()
w = torch.randn(N, d, device="cuda") / d ** 0.5
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
L = _lib.lib()
for k in (1, 2):
    q = K.expert_quota(2.0, T, k, N)
    dec = K.gate_topk(x, w, k, q)
    buf = K.dispatch(x, dec.indices, dec.slots, N, q)
    for mult in (1, 2, 4, 8, 16, 0):
        if mult == 0:
            ctypes.c_int.in_dll(L, "scmoe_dispatch_force_ldst").value = 1
        else:
            ctypes.c_int.in_dll(L, "scmoe_dispatch_force_ldst").value = 0
            ctypes.c_int.in_dll(L, "scmoe_dispatch_bulk_ctas_per_sm").value = mult
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            K.dispatch(x, dec.indices, dec.slots, N, q, out=buf)
            with torch.cuda.graph(g, stream=s):
                K.dispatch(x, dec.indices, dec.slots, N, q, out=buf)
        torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
        ts = []
        for i in range(12):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); g.replay(); b.record(); torch.cuda.synchronize()
            if i > 1: ts.append(a.elapsed_time(b) * 1e3)
        print(f"k={k} {'ldst' if mult == 0 else f'bulk x{mult}'}: {statistics.median(ts):.1f} us")
