"""Expert parallelism over peer memory (csrc/dispatch.cu K9/K10,
paper_2404_05019_b200/ep_p2p.py), checked on one B200 with VIRTUAL ranks:
G ranks' symmetric buffers live on the same GPU and every rank's peer
tables point at the others' buffers, exactly the addressing the NVLink path
uses across GPUs.  Per rank, the EP result must equal the single-GPU layer on
that rank's tokens (all experts local) bit for bit — routing, quota and slots
are per rank (gating.py:134-135), the grouped FFN rows are identical.

Covered: world 2 / 4, 1 and 2 experts per rank, top-1 ScMoE (SE + CG
combine) and top-2, pull-form combine (rows read from the owner's y) and
push-form return (owner stores rows into the source's back buffer), the
fused return (the owner's GEMM2 epilogue stores rows into the sources' back
buffers), several
calls in a row (epoch flags advance, buffers reused), a CUDA-graph capture of
the whole sequence replayed with new inputs, and a one-rank symmetric-memory
rendezvous over NCCL."""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu
P = None


def setup_module(module):
    global P
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2404_05019_b200 as pkg
    P = pkg
    torch.cuda.set_device(0)


def _local_experts(layer, r, e_l):
    from paper_2404_05019_b200.layers import RoutedExperts
    ex = RoutedExperts(e_l, layer.d_model, layer.d_hidden, dtype=torch.bfloat16, device="cuda")
    with torch.no_grad():
        for name in ("w1t", "b1", "w2t", "b2"):
            getattr(ex, name).copy_(getattr(layer.experts, name)[r * e_l:(r + 1) * e_l])
    return ex


def _run_ep(layer, xs, srcs, world, e_l, form, mode):
    """One EP forward of every virtual rank; returns the per-rank outputs."""
    from paper_2404_05019_b200.ep_p2p import PeerExchange
    decs = [layer.route(s) for s in srcs]
    cap = decs[0].capacity
    if not hasattr(layer, "_vx") or layer._vx[0].capacity != cap:
        layer._vx = PeerExchange.virtual(world, e_l, cap, layer.d_model, torch.bfloat16, "cuda")
        layer._vex = [_local_experts(layer, r, e_l) for r in range(world)]
    vx, vex = layer._vx, layer._vex
    for r in range(world):
        vx[r].dispatch(srcs[r], decs[r].indices, decs[r].slots, decs[r].counts,
                       max_ctas=(32 if r % 2 else 0))
    for r in range(world):
        if form == "fused":
            vx[r].expert_ffn_to_peers(vex[r])
            continue
        vx[r].expert_ffn(vex[r], signal=(form == "pull"))
        if form == "push":
            vx[r].push_back(max_ctas=16)
    outs = []
    for r in range(world):
        std = not hasattr(layer, "shared")
        kw = {} if std else dict(se_out=layer.shared(xs[r]), mode=layer.combine_mode,
                                 x_cur=xs[r], w_cg=layer.w_cg)
        if form == "pull":
            outs.append(vx[r].combine(decs[r].indices, decs[r].slots, decs[r].weights, **kw))
        else:
            outs.append(vx[r].combine_local(decs[r].indices, decs[r].slots, decs[r].weights, **kw))
    return outs


def _layer(kind, d, h, n, mode):
    g = torch.Generator(device="cuda").manual_seed(11)
    if kind == "scmoe":
        return P.ScMoELayer(d, h, n, combine_mode=mode, capacity_factor=1.25,
                            dtype=torch.bfloat16, generator=g)
    return P.Top2MoELayer(d, h, n, capacity_factor=1.0, dtype=torch.bfloat16, generator=g)


@pytest.mark.parametrize("world,e_l", [(2, 1), (2, 2), (4, 1), (4, 2)])
@pytest.mark.parametrize("kind,mode", [("scmoe", "direct_add"), ("scmoe", "cg2"), ("top2", None)])
@pytest.mark.parametrize("form", ["pull", "push", "fused"])
def test_p2p_ep_equals_local(world, e_l, kind, mode, form):
    T, d, h = 300, 128, 256
    layer = _layer(kind, d, h, world * e_l, mode)
    for call in range(3):        # epochs 1..3: flags advance, buffers are reused
        g = torch.Generator(device="cuda").manual_seed(100 * call + world)
        xs = [torch.randn(T, d, device="cuda", generator=g).bfloat16() for _ in range(world)]
        srcs = [torch.randn(T, d, device="cuda", generator=g).bfloat16() for _ in range(world)]
        with torch.no_grad():
            if kind == "scmoe":
                outs = _run_ep(layer, xs, srcs, world, e_l, form, mode)
                refs = [layer(xs[r], srcs[r])[0] for r in range(world)]
            else:        # top-2 routes and combines the same tokens
                outs = _run_ep(layer, srcs, srcs, world, e_l, form, mode)
                refs = [layer(srcs[r])[0] for r in range(world)]
        torch.cuda.synchronize()
        for r in range(world):
            assert torch.equal(outs[r], refs[r]), (call, r)
    assert all(int(v.epoch[0]) == 3 for v in layer._vx)


def test_p2p_ep_cuda_graph_replay():
    """The dispatch / wait / FFN / return / combine sequence of 2 virtual ranks
    captured once and replayed with fresh inputs: the device-side epoch makes
    every replay wait for its own flags."""
    world, e_l, T, d, h = 2, 2, 256, 128, 256
    layer = _layer("scmoe", d, h, world * e_l, "direct_add")
    xs = [torch.randn(T, d, device="cuda").bfloat16() for _ in range(world)]
    srcs = [torch.randn(T, d, device="cuda").bfloat16() for _ in range(world)]
    with torch.no_grad():
        _run_ep(layer, xs, srcs, world, e_l, "push", None)        # warm-up, epoch 1
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(gr, stream=s):
                outs = _run_ep(layer, xs, srcs, world, e_l, "push", None)
        torch.cuda.current_stream().wait_stream(s)
        for it in range(3):
            g = torch.Generator(device="cuda").manual_seed(7 + it)
            for r in range(world):
                xs[r].copy_(torch.randn(T, d, device="cuda", generator=g))
                srcs[r].copy_(torch.randn(T, d, device="cuda", generator=g))
            gr.replay()
            torch.cuda.synchronize()
            for r in range(world):
                ref = layer(xs[r], srcs[r])[0]
                assert torch.equal(outs[r], ref), (it, r)
    assert all(int(v.epoch[0]) == 1 + 3 for v in layer._vx)   # warm-up + 3 replays


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_p2p_symmetric_memory_one_rank():
    """PeerExchange.from_group over a one-rank NCCL group (torch symmetric
    memory for allocation + rendezvous); the exchange itself is our kernels."""
    import torch.distributed as dist
    from paper_2404_05019_b200.ep_p2p import PeerExchange
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0,
                                world_size=1, device_id=torch.device("cuda", 0))
    try:
        T, d, h, n = 512, 128, 256, 4
        layer = _layer("scmoe", d, h, n, "cg1")
        x = torch.randn(T, d, device="cuda").bfloat16()
        src = torch.randn(T, d, device="cuda").bfloat16()
        with torch.no_grad():
            dec = layer.route(src)
            px = PeerExchange.from_group(dist.group.WORLD, n, dec.capacity, d, torch.bfloat16,
                                         "cuda")
            for _ in range(2):
                px.dispatch(src, dec.indices, dec.slots, dec.counts)
                px.expert_ffn(layer.experts, signal=False)
                px.push_back()
                out = px.combine_local(dec.indices, dec.slots, dec.weights,
                                       se_out=layer.shared(x), mode="cg1", x_cur=x,
                                       w_cg=layer.w_cg)
                ref = layer(x, src)[0]
                torch.cuda.synchronize()
                assert torch.equal(out, ref)
    finally:
        if own:
            dist.destroy_process_group()
