"""Why is the standalone ScMoE layer slower than top-2 on the p2p EP path?
One-rank NCCL group on one GPU (the EP code path with a local peer table):
CUPTI kernel list of one layer call per arm, and CUDA-event times (eager and
graphed), next to the local (non-EP) layer.

    python scripts/ep_layer_probe.py"""
import os
import socket
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from torch.profiler import ProfilerActivity, profile

with socket.socket() as s_:
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
import paper_2404_05019_b200 as P
from paper_2404_05019_b200.runtime import CapturedStep

T, d, h, N = 16384, 2048, 8192, 8
x = torch.randn(T, d, device="cuda").bfloat16()
src = torch.randn(T, d, device="cuda").bfloat16()
arms = {}
for ep in (False, True):
    g = dist.group.WORLD if ep else None
    sc = P.ScMoELayer(d, h, N, dtype=torch.bfloat16, ep_group=g,
                      generator=torch.Generator(device="cuda").manual_seed(1))
    t2 = P.Top2MoELayer(d, h, N, dtype=torch.bfloat16, ep_group=g,
                        generator=torch.Generator(device="cuda").manual_seed(1))
    if ep:
        sc.ep_backend = t2.ep_backend = "p2p"
    arms[f"scmoe{'_ep' if ep else ''}"] = lambda xx, m=sc: m(xx, src)[0]
    arms[f"top2{'_ep' if ep else ''}"] = lambda xx, m=t2: m(xx)[0]


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / n)
    return statistics.median(ts)


with torch.no_grad():
    for name, fn in arms.items():
        eager = timeit(lambda: fn(x))
        g = CapturedStep(fn, [x])
        graph = timeit(lambda: g.replay())
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            g.replay()
            torch.cuda.synchronize()
        ks = [(e.name.split("(")[0][-60:], (getattr(e, "device_time_total", 0.0) or e.cuda_time_total))
              for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
        print(f"== {name}: eager {eager:.3f} ms  graph {graph:.3f} ms")
        for k, us in ks:
            print(f"   {us:8.1f} us  {k}")
dist.destroy_process_group()
