"""The expert-parallel path over a real NCCL communicator of one rank: the
side-stream all-to-alls, cross-stream events, chunked exchanges and the
comm-span recording all run on the GPU (a one-rank all-to-all is a local
copy), and the results must equal the single-GPU path bit for bit.  The
multi-rank exchange logic itself is covered over gloo in test_ep_gloo.py."""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu
P = None


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def setup_module(module):
    global P
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import torch.distributed as dist
    import paper_2404_05019_b200 as pkg
    P = pkg
    if not dist.is_initialized():
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0,
                                world_size=1, device_id=torch.device("cuda", 0))


def teardown_module(module):
    import torch.distributed as dist
    if dist.is_initialized():
        dist.destroy_process_group()


@pytest.mark.parametrize("variant,chunks", [("scmoe", 1), ("scmoe", 2), ("standard", 1),
                                            ("standard", 3)])
def test_ep_path_equals_local(variant, chunks):
    import torch.distributed as dist
    from paper_2404_05019_b200.timeline import Recorder, comm_overlap_fraction
    T, d, h, N = 1024, 256, 512, 8
    kw = dict(variant=variant, k_routed=1 if variant == "scmoe" else 2,
              shortcut_pos="pos2" if variant == "scmoe" else None, n_heads=4, seq_len=256,
              capacity_factor=1.25, dtype=torch.bfloat16, chunks=chunks)
    loc = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(2), **kw)
    epb = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(2),
                           ep_group=dist.group.WORLD, **kw)
    x = torch.randn(T, d, device="cuda").bfloat16()
    with torch.no_grad():
        a, _, _ = loc(x)
        rec = Recorder()
        b, _, _ = epb(x, recorder=rec)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    spans = rec.spans()
    comm = [s for s in spans if s.stream == "comm"]
    assert len(comm) == 2 * chunks          # dispatch + combine per chunk
    assert 0.0 <= comm_overlap_fraction(spans) <= 1.0


def test_ep_calibrate_and_train_step():
    import torch.distributed as dist
    blk = P.ScMoEBlockPair(256, 512, 8, variant="scmoe", shortcut_pos="pos2", n_heads=4,
                           seq_len=256, dtype=torch.bfloat16, ep_group=dist.group.WORLD,
                           generator=torch.Generator(device="cuda").manual_seed(3))
    x = torch.randn(1024, 256, device="cuda").bfloat16()
    with torch.no_grad():
        ch = blk.calibrate(x)
    assert 0 <= ch.slot <= 3 and blk.last_costs.t_disp >= 0
    blk.requires_grad_(True)
    l0 = float(blk.train_step(x, lr=1e-3))
    l1 = float(blk.train_step(x, lr=1e-3))
    assert l1 < l0


@pytest.mark.parametrize("variant,slot,ret", [("scmoe", 0, "fused"), ("scmoe", 2, "push"),
                                              ("standard", None, "fused"), ("scmoe", 1, "push")])
def test_ep_p2p_backend_equals_local(variant, slot, ret):
    """ep_backend="p2p": dispatch and return trip are our peer-memory kernels
    on the side stream (symmetric memory over the one-rank group); repeated
    forwards reuse the buffers (epoch flags)."""
    import torch.distributed as dist
    from paper_2404_05019_b200.timeline import Recorder
    T, d, h, N = 1024, 256, 512, 8
    kw = dict(variant=variant, k_routed=1 if variant == "scmoe" else 2,
              shortcut_pos="pos2" if variant == "scmoe" else None, n_heads=4, seq_len=256,
              capacity_factor=1.25, dtype=torch.bfloat16)
    loc = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(2), **kw)
    epb = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(2),
                           ep_group=dist.group.WORLD, ep_backend="p2p", p2p_return=ret, **kw)
    if slot is not None:
        epb.slot = loc.slot = slot
    for it in range(3):
        x = torch.randn(T, d, device="cuda").bfloat16()
        with torch.no_grad():
            a, _, _ = loc(x)
            rec = Recorder()
            b, _, _ = epb(x, recorder=rec)
        torch.cuda.synchronize()
        assert torch.equal(a, b), it
        comm = [s for s in rec.spans() if s.stream == "comm"]
        assert len(comm) == (1 if ret == "fused" else 2)   # fused: return inside GEMM2


@pytest.mark.parametrize("variant", ["scmoe", "standard"])
def test_ep_training_step_equals_local(variant):
    """Training under expert parallelism: the exchanges (and their backward,
    the reverse exchanges) run on the comm stream; on one rank the gradients
    and the updated weights equal the local block's bit for bit."""
    import torch.distributed as dist
    T, d, h, N = 512, 128, 256, 4
    kw = dict(variant=variant, k_routed=1 if variant == "scmoe" else 2,
              shortcut_pos="pos2" if variant == "scmoe" else None, n_heads=4, seq_len=128,
              capacity_factor=1.25, dtype=torch.bfloat16)
    loc = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(6), **kw)
    epb = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(6),
                           ep_group=dist.group.WORLD, **kw)
    loc.requires_grad_(True)
    epb.requires_grad_(True)
    x = torch.randn(T, d, device="cuda").bfloat16()
    for it in range(2):
        la = loc.train_step(x, lr=1e-3)
        lb = epb.train_step(x, lr=1e-3)
        torch.cuda.synchronize()
        assert torch.equal(la, lb), it
    for (na, pa), (nb, pb) in zip(loc.named_parameters(), epb.named_parameters()):
        assert torch.equal(pa, pb), na


@pytest.mark.parametrize("variant,chunks,ret", [("scmoe", 2, "fused"), ("standard", 3, "fused"),
                                                ("scmoe", 4, "push"), ("standard", 2, "push")])
def test_ep_p2p_chunked_equals_local(variant, chunks, ret):
    """Chunked pipelining on the p2p backend (distsim.py:277-300, 358-364):
    one peer-memory exchange per chunk with its own flags and epoch, chunk
    c's expert FFN starts when chunk c's rows landed, the return rows land in
    a chunk-major back buffer and one combine gathers them.  Equal to the
    local unchunked block bit for bit over repeated eager calls and over CUDA
    graph replays with fresh inputs."""
    import torch.distributed as dist
    from paper_2404_05019_b200.runtime import CapturedStep
    from paper_2404_05019_b200.timeline import Recorder
    T, d, h, N = 1024, 256, 512, 8
    kw = dict(variant=variant, k_routed=1 if variant == "scmoe" else 2,
              shortcut_pos="pos2" if variant == "scmoe" else None, n_heads=4, seq_len=256,
              capacity_factor=1.25, dtype=torch.bfloat16)
    loc = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(2), **kw)
    epb = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(2),
                           ep_group=dist.group.WORLD, ep_backend="p2p", p2p_return=ret,
                           chunks=chunks, **kw)
    for it in range(2):
        x = torch.randn(T, d, device="cuda").bfloat16()
        with torch.no_grad():
            a, _, _ = loc(x)
            rec = Recorder()
            b, _, _ = epb(x, recorder=rec)
        torch.cuda.synchronize()
        assert torch.equal(a, b), it
        comm = [s for s in rec.spans() if s.stream == "comm"]
        assert len(comm) == chunks * (1 if ret == "fused" else 2)
    x = torch.randn(T, d, device="cuda").bfloat16()
    with torch.no_grad():
        g = CapturedStep(lambda xx: epb(xx)[0], [x])
        for it in range(3):
            x = torch.randn(T, d, device="cuda").bfloat16()
            out = g(x)
            ref, _, _ = loc(x)
            torch.cuda.synchronize()
            assert torch.equal(out, ref), it


@pytest.mark.parametrize("backend", ["nccl", "p2p"])
@pytest.mark.parametrize("constraint", [True, False])
def test_ep_dgmoe_equals_local(backend, constraint):
    """DGMoE (dual gating, arch.py:507-533) under expert parallelism: both
    gatings' rows travel as one 2T-row routing with 2*cap slots per expert;
    the block output and both decisions equal the local block's bit for bit."""
    import torch.distributed as dist
    T, d, h, N = 1024, 256, 512, 8
    kw = dict(variant="dgmoe", n_heads=4, seq_len=256, capacity_factor=1.0,
              dtype=torch.bfloat16, dgmoe_constraint=constraint)
    loc = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(8), **kw)
    epb = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(8),
                           ep_group=dist.group.WORLD, ep_backend=backend, **kw)
    for it in range(2):
        x = torch.randn(T, d, device="cuda").bfloat16()
        with torch.no_grad():
            a, (dca, dpa), _ = loc(x)
            b, (dcb, dpb), _ = epb(x)
        torch.cuda.synchronize()
        assert torch.equal(dca.indices, dcb.indices) and torch.equal(dpa.slots, dpb.slots)
        assert int(dpa.dropped.sum()) > 0 or int(dca.dropped.sum()) > 0   # cf 1.0 drops
        assert torch.equal(a, b), it
