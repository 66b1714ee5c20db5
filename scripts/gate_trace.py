"""Per-CTA timeline of the tensor-core gate (build_ab/libscmoe_gtrace.so, built
with -DSCMOE_GATE_TRACE): entry, first stage landed, last tile published,
grid-wide wait done, exit — in us from the earliest CTA entry.

    SCMOE_LIB=build_ab/libscmoe_gtrace.so python scripts/gate_trace.py [T]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2404_05019_b200 import kernels as K, _lib
T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
d, N = 2048, 8
w = torch.randn(N, d, device="cuda") / d ** 0.5
ws = K.gate_split_weights(w)
x = torch.randn(T, d, device="cuda").bfloat16()
quota = K.expert_quota(2.0, T, 1, N)
flush = torch.ones(128 * 1024 * 1024, device="cuda")
lib = _lib.lib()
fn = lib.scmoe_debug_gate_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
n16 = (T + 15) // 16
ctas = min(n16, torch.cuda.get_device_properties(0).multi_processor_count)
tiles = ctas * ((n16 + ctas - 1) // ctas + 3) // 4     # sub-tiles of <= 4 row tiles per CTA
for rep in range(4):
    flush.sum()
    torch.cuda.synchronize()
    K.gate_topk(x, w, 1, quota, w_split=ws)
    torch.cuda.synchronize()
buf = np.zeros((ctas, 20), dtype=np.uint64)
assert fn(buf.ctypes.data, ctas) == 0
t0 = buf[:, 0].min()
r = (buf.astype(np.int64) - int(t0)) / 1e3
names = ["entry", "stage0", "published", "wait_done", "exit", "rt_got", "rt_done", "mma_done",
         "lempty_ok", "logits_out", "rp_a", "rp_sync1", "rp_b", "rp_sync2",
         "rp_h_loaded", "rp_logits_st", "rp_topk_w", "rp_softmax"]
for i, n in enumerate(names):
    col = r[:, i]
    print(f"{n:10s} min {col.min():7.2f}  median {np.median(col):7.2f}  max {col.max():7.2f} us")
fs = lib.scmoe_debug_gate_stages
fs.argtypes = [ctypes.c_void_p, ctypes.c_int]
st = np.zeros((ctas, 32), dtype=np.uint64)
assert fs(st.ctypes.data, ctas) == 0
nst = min(32, ((tiles + ctas - 1) // ctas) * ((d + 255) // 256))
sr = (st[:, :nst].astype(np.int64) - int(t0)) / 1e3
print("stage landed (median over CTAs, us):", " ".join(f"{v:.2f}" for v in np.median(sr, axis=0)))
