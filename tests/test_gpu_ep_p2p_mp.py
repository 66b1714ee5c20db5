"""The peer-memory expert-parallel path across PROCESSES: two ranks (two
processes) share the one B200 of the test box, their symmetric buffers are
mapped into each other through CUDA IPC (torch symmetric memory over a gloo
group — allocation and handle exchange only), and every byte of the exchange
is moved by our kernels with system-scope fences and epoch flags, exactly as
across NVLink.  Each rank's block-pair output must equal a single-process
block holding all experts, on that rank's tokens, bit for bit (per-rank
routing and quota, gating.py:134-135)."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, variant, q, chunks=1):
    import sys
    sys.path.insert(0, ROOT)
    try:
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        import paper_2404_05019_b200 as P
        T, d, h, N = 512, 256, 512, 4 * world
        kw = dict(variant=variant, k_routed=2 if variant == "standard" else 1,
                  shortcut_pos="pos2" if variant == "scmoe" else None, n_heads=4, seq_len=256,
                  capacity_factor=1.25, dtype=torch.bfloat16)
        loc = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(5),
                               **kw)
        epb = P.ScMoEBlockPair(d, h, N, ep_group=dist.group.WORLD, ep_backend="p2p",
                               chunks=chunks, **kw)
        e_l = N // world
        with torch.no_grad():
            src = dict(loc.named_parameters())
            for name, p in epb.named_parameters():
                full = src[name]
                if name.startswith("moe.experts."):
                    p.copy_(full[rank * e_l:(rank + 1) * e_l])
                else:
                    p.copy_(full)
        for it in range(3):
            g = torch.Generator(device="cuda").manual_seed(1000 * it + rank)
            x = torch.randn(T, d, device="cuda", generator=g).bfloat16()
            with torch.no_grad():
                a, _, _ = loc(x)
                b, _, _ = epb(x)
            torch.cuda.synchronize()
            if not torch.equal(a, b):
                raise AssertionError(f"rank {rank} call {it}: max diff "
                                     f"{(a.float() - b.float()).abs().max().item()}")
        # the standalone layer module (moe_shared / moe_standard drop-in) on the
        # p2p backend, same weights as the local block's layer
        epl = epb.moe
        with torch.no_grad():
            x = torch.randn(T, d, device="cuda", generator=torch.Generator(device="cuda")
                            .manual_seed(7 + rank)).bfloat16()
            if variant in ("scmoe", "dgmoe"):
                a = loc.moe(x, x.flip(0))[0]
                b = epl(x, x.flip(0))[0]
            else:
                a = loc.moe(x)[0]
                b = epl(x)[0]
        torch.cuda.synchronize()
        if not torch.equal(a, b):
            raise AssertionError(f"rank {rank}: layer-level p2p differs")
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("variant,chunks", [("scmoe", 1), ("standard", 1), ("scmoe", 2),
                                            ("standard", 3), ("dgmoe", 1)])
def test_p2p_ep_two_processes(variant, chunks):
    """chunks > 1: chunked pipelining across the processes (one exchange per
    chunk, chunk-major return rows)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, variant, q, chunks)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, msg = q.get(timeout=240)
        res[r] = msg
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
