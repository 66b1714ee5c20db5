"""Expert-parallel TRAINING across two processes (world 2): two ranks share
the test box's GPU over a gloo group (the exchange code is torch.distributed
all-to-all, the same calls NCCL runs between GPUs).  Each rank trains on its
own token slice; the gradients after `train_step`'s reduction must equal the
gradients of the mean of the per-rank objectives, (1/G) sum_r loss_r,
computed by one process holding every expert (grad.py:52-67 per slice):

  * replicated parameters (gate, shared expert, backbone): averaged;
  * routed experts (sharded): the owner's weight-gradient GEMM sums every
    source rank's rows, then divides by G — the same mean.

bf16 with a different summation order: |g_ep - g_ref| <= rtol (|g_ref| +
max|g_ref|) per tensor, rtol 2e-2."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RTOL = 2e-2


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, variant, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        import paper_2404_05019_b200 as P
        T, d, h, N = 512, 128, 256, 2 * world
        kw = dict(variant=variant, k_routed=1 if variant == "scmoe" else 2,
                  shortcut_pos="pos2" if variant == "scmoe" else None, n_heads=2, seq_len=128,
                  capacity_factor=1.25, dtype=torch.bfloat16)
        loc = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(3),
                               **kw)
        epb = P.ScMoEBlockPair(d, h, N, ep_group=dist.group.WORLD, ep_backend="nccl", **kw)
        e_l = N // world
        with torch.no_grad():
            src = dict(loc.named_parameters())
            for name, p in epb.named_parameters():
                full = src[name]
                p.copy_(full[rank * e_l:(rank + 1) * e_l] if name.startswith("moe.experts.")
                        else full)
        loc.requires_grad_(True)
        epb.requires_grad_(True)
        xs = [torch.randn(T, d, device="cuda",
                          generator=torch.Generator(device="cuda").manual_seed(50 + r)).bfloat16()
              for r in range(world)]
        tgt = [torch.randn(T, d, device="cuda",
                           generator=torch.Generator(device="cuda").manual_seed(80 + r)).bfloat16()
               for r in range(world)]
        # expert-parallel step on my slice (reduction inside train_step)
        epb.train_step(xs[rank], target=tgt[rank], update=False)
        # reference: every slice through the all-expert block, mean of the losses
        for p in loc.parameters():
            p.grad = None
        total = 0.0
        for r in range(world):
            out, _, aux = loc(xs[r])
            loss = (out.float() - tgt[r].float()).pow(2).sum() / T + 0.01 * aux
            total = total + loss / world
        total.backward()
        torch.cuda.synchronize()
        ref = dict(loc.named_parameters())
        bad = []
        for name, p in epb.named_parameters():
            r = ref[name].grad
            if name.startswith("moe.experts."):
                r = r[rank * e_l:(rank + 1) * e_l]
            if p.grad is None or r is None:
                if (p.grad is None) != (r is None):
                    bad.append(f"{name}: grad presence differs")
                continue
            a, b = p.grad.double(), r.double()
            bound = RTOL * (b.abs() + b.abs().max() + 1e-30)
            worst = float(((a - b).abs() / bound).max())
            if worst > 1.0:
                bad.append(f"{name}: worst err/bound {worst:.3g}")
        if bad:
            raise AssertionError(f"rank {rank}: " + "; ".join(bad))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("variant", ["scmoe", "standard"])
def test_ep_training_gradients_two_processes(variant):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, variant, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, msg = q.get(timeout=300)
        res[r] = msg
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
