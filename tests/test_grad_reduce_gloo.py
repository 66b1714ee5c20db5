"""Gradient reduction of expert-parallel training over world_size 2 (gloo, CPU).

The objective of G ranks training together is the mean of the per-rank
objectives (each rank runs the reference's compute_loss on its slice,
grad.py:52-67).  Replicated parameters hold d loss_r / dp on rank r and are
averaged; a sharded routed expert's gradient is already summed over the
source ranks by its owner's weight-gradient GEMM (the reverse exchange brings
every rank's dy to the owner), so it is divided by G, not all-reduced.
Without expert parallelism the experts are replicas and are averaged too."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from torch import nn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _Toy(nn.Module):
    def __init__(self):
        super().__init__()
        self.attn = nn.Linear(3, 2, bias=False)
        self.moe = nn.Module()
        self.moe.experts = nn.Module()
        self.moe.experts.w1t = nn.Parameter(torch.zeros(2, 4))
        self.moe.shared = nn.Module()
        self.moe.shared.w1t = nn.Parameter(torch.zeros(4))


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        from paper_2404_05019_b200.training import allreduce_replicated_grads
        for sharded in (True, False):
            m = _Toy()
            for i, p in enumerate(m.parameters()):
                p.grad = torch.full_like(p, float(10 * (rank + 1) + i))
            allreduce_replicated_grads(m, experts_sharded=sharded)
            for i, (n, p) in enumerate(m.named_parameters()):
                mine = 10 * (rank + 1) + i
                mean = sum(10 * (r + 1) + i for r in range(world)) / world
                want = mine / world if (sharded and ".experts." in f".{n}") else mean
                assert torch.allclose(p.grad, torch.full_like(p, want)), (n, sharded, p.grad)
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover - surfaced through the queue
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_grad_reduction_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=110) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert results == {0: "ok", 1: "ok"}, results
