"""Can the expert-parallel training step (NCCL exchange + replicated-grad
all-reduce) be captured in a CUDA graph?  One-rank NCCL group (or torchrun
ranks): capture train_step, replay, compare the loss with eager steps on a
twin block, time both."""
import os, sys, socket
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
if "RANK" not in os.environ:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0)); port = sk.getsockname()[1]
    os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
import paper_2404_05019_b200 as P
from paper_2404_05019_b200.runtime import CapturedStep
T, d, h, N = 18432, 384, 1536, 8
def make():
    return P.ScMoEBlockPair(d, h, N, variant="scmoe", shortcut_pos="pos2", n_heads=12, seq_len=144,
                            capacity_factor=1.25, dtype=torch.bfloat16, ep_group=dist.group.WORLD,
                            generator=torch.Generator(device="cuda").manual_seed(1)).requires_grad_(True)
x = torch.randn(T, d, device="cuda", generator=torch.Generator(device="cuda").manual_seed(2)).bfloat16()
a, b = make(), make()
eager = [float(a.train_step(x, lr=1e-3)) for _ in range(4)]
g = CapturedStep(lambda xx: b.train_step(xx, lr=1e-3), [x], warmup=3)
graph = [float(g.replay()) for _ in range(1)]
print("eager losses", eager, "graph loss after 3 warmup + 1 replay", graph)
torch.cuda.synchronize()
import time
for name, fn in (("eager", lambda: a.train_step(x, lr=1e-3)), ("graph", g.replay)):
    for _ in range(3): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(10): fn()
    torch.cuda.synchronize()
    print(name, f"{(time.perf_counter() - t0) / 10 * 1e3:.3f} ms/step")
dist.destroy_process_group()
