"""Layer / block parity against the float64 oracle (pinned to the reference).

Tolerance (north star): rtol 1e-4 in fp32, 2e-2 in bf16, checked as
|gpu - ref| <= atol + rtol*|ref| with atol = rtol * max|ref| (SURVEY §7,
hard part 2: a pure elementwise rtol fails near zero even for exact fp32).
Routing is compared bit-exactly on identical logits, and the outputs with the
GPU's routing pinned into the oracle (MoEReplay semantics, arch.py:395-402).
"""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import scmoe_oracle as O

pytestmark = pytest.mark.gpu

P = None
RTOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


def setup_module(module):
    global P
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2404_05019_b200 as pkg
    P = pkg


def _check(gpu, ref, rtol, what):
    ok, worst = O.allclose_scaled(gpu, ref, rtol)
    assert ok, f"{what}: worst error / bound = {worst:.3g} (rtol {rtol})"


def _check_routing(dec, src_logits_np, k, cf):
    n = src_logits_np.shape[1]
    ref = O.apply_capacity(O.select_topk(src_logits_np, k), cf, n, src_logits_np.shape[0])
    np.testing.assert_array_equal(dec.indices.long().cpu().numpy(), ref.indices)
    np.testing.assert_array_equal(dec.dropped.cpu().numpy(), ref.dropped)


def _t(a, dtype):
    return torch.as_tensor(np.asarray(a), device="cuda").to(dtype).contiguous()


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("mode", ["direct_add", "cg1", "cg2"])
def test_scmoe_layer_cfg1(dtype, mode):
    """BASELINE configs[0] layer: d=256, h=1024, N=8, top-1 + SE, cf=1.0, T=512."""
    T, d, h, N, cf = 512, 256, 1024, 8, 1.0
    rng = O.Rng(11)
    pp = O.init_pair(d, h, N, rng.spawn(0), variant="scmoe", combine_mode=mode)
    x_cur = rng.spawn(1).normal((T, d))
    src = rng.spawn(2).normal((T, d))
    layer = P.ScMoELayer.from_reference(pp.moe, P.CapacityConfig(cf), dtype=dtype)
    xc, xs = _t(x_cur, dtype), _t(src, dtype)
    out, dec, aux = layer(xc, xs)
    torch.cuda.synchronize()
    _check_routing(dec, dec.logits.double().cpu().numpy(), 1, cf)
    ref_out, ref_dec, ref_aux = O.moe_shared(
        xc.double().cpu().numpy(), pp.moe, cf, 1, routed_src=xs.double().cpu().numpy(),
        pinned_indices=dec.indices.long().cpu().numpy(), pinned_dropped=dec.dropped.cpu().numpy())
    _check(out.double().cpu().numpy(), ref_out, RTOL[dtype], f"moe_shared {mode} {dtype}")
    assert float(aux) == pytest.approx(ref_aux, rel=RTOL[dtype], abs=1e-4)
    # unpinned oracle routing agrees on (almost) every token
    free = O.moe_shared(xc.double().cpu().numpy(), pp.moe, cf, 1,
                        routed_src=xs.double().cpu().numpy())[1]
    agree = (free.indices == dec.indices.long().cpu().numpy()).mean()
    assert agree > 0.98


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("cf", [2.0, 0.6])
def test_top2_layer(dtype, cf):
    T, d, h, N = 384, 128, 512, 8
    rng = O.Rng(5)
    pp = O.init_pair(d, h, N, rng.spawn(0), variant="standard", k=2)
    x = rng.spawn(1).normal((T, d))
    layer = P.Top2MoELayer.from_reference(pp.moe, P.CapacityConfig(cf), dtype=dtype)
    xt = _t(x, dtype)
    out, dec, aux = layer(xt)
    torch.cuda.synchronize()
    _check_routing(dec, dec.logits.double().cpu().numpy(), 2, cf)
    ref_out, _, ref_aux = O.moe_standard(
        xt.double().cpu().numpy(), pp.moe, cf, 2,
        pinned_indices=dec.indices.long().cpu().numpy(), pinned_dropped=dec.dropped.cpu().numpy())
    _check(out.double().cpu().numpy(), ref_out, RTOL[dtype], f"moe_standard cf={cf} {dtype}")
    assert float(aux) == pytest.approx(ref_aux, rel=RTOL[dtype], abs=1e-4)
    if cf < 1:
        assert dec.dropped.any()


def test_noise_and_replay():
    T, d, h, N = 200, 64, 128, 4
    rng = O.Rng(2)
    pp = O.init_pair(d, h, N, rng.spawn(0), variant="scmoe", combine_mode="cg1", noise_enabled=True)
    x = rng.spawn(1).normal((T, d))
    eps = rng.spawn(2).normal((T, N))
    layer = P.ScMoELayer.from_reference(pp.moe, P.CapacityConfig(1.0), dtype=torch.float32)
    xt = _t(x, torch.float32)
    out, dec, _ = layer(xt, xt, eps=_t(eps, torch.float32))
    ref_out, _, _ = O.moe_shared(x, pp.moe, 1.0, 1, eps=eps,
                                 pinned_indices=dec.indices.long().cpu().numpy(),
                                 pinned_dropped=dec.dropped.cpu().numpy())
    _check(out.double().cpu().numpy(), ref_out, 1e-4, "noisy gate")
    # replay with pinned routing reproduces the forward bit for bit
    rep = P.MoEReplay(eps=eps, indices=dec.indices.long().cpu().numpy(),
                      dropped=dec.dropped.cpu().numpy())
    out2, dec2, _ = layer(xt, xt, replay=rep)
    assert torch.equal(out, out2)


def _pair_ns(pp, cfg):
    prev = SimpleNamespace(attn=pp.attn_prev, feed=pp.mlp_prev)
    cur = SimpleNamespace(attn=pp.attn_cur, feed=pp.moe)
    return cfg, prev, cur


@pytest.mark.parametrize("variant,pos,mode,k", [
    ("scmoe", "pos2", "direct_add", 1), ("scmoe", "pos1", "cg2", 1), ("scmoe", "pos3", "cg1", 1),
    ("shared", None, "direct_add", 1), ("standard", None, "direct_add", 2),
    ("scmoe", "pos2", "direct_add", 2)])
def test_block_pair_cfg1_fp32(variant, pos, mode, k):
    """BASELINE configs[0]: the tiny block pair (d=256, N=8, cf=1.0, 4x128 tokens), fp32."""
    T, d, h, N, cf = 512, 256, 1024, 8, 1.0
    pp = O.init_pair(d, h, N, O.Rng(0).spawn(0), variant=variant, k=k, combine_mode=mode)
    tokens = O.Rng(0).spawn(1).normal((T, d))
    cfg = SimpleNamespace(d_model=d, d_hidden=h, n_experts=N, variant=variant, shortcut_pos=pos,
                          k_routed=k, combine_mode=mode, capacity_factor=cf, noise_enabled=False,
                          pre_layernorm=False)
    blk = P.ScMoEBlockPair.from_reference(*_pair_ns(pp, cfg), dtype=torch.float32)
    out, dec, aux, taps = blk(_t(tokens, torch.float32), return_taps=True)
    torch.cuda.synchronize()
    ref_out, ref_dec, ref_aux, ref_taps = O.block_pair_forward(
        pp, tokens, variant, pos, cf, k, pinned_indices=dec.indices.long().cpu().numpy(),
        pinned_dropped=dec.dropped.cpu().numpy())
    for name in ("h_mh_prev", "h_mlp_prev", "h_mh_cur"):
        _check(taps[name].double().cpu().numpy(), ref_taps[name], 1e-4, name)
    _check(out.double().cpu().numpy(), ref_out, 1e-4, f"block pair {variant}/{pos}/{mode}")
    assert float(aux) == pytest.approx(ref_aux, rel=1e-4, abs=1e-5)


def test_block_pair_cfg1_matches_reference_golden(golden_dir):
    """Against the reference's own output for configs[0] (tests/golden/cfg1_case.npz)."""
    import os
    z = np.load(os.path.join(golden_dir, "cfg1_case.npz"))
    T, d, h, N = 512, 256, 1024, 8
    pp = O.init_pair(d, h, N, O.Rng(0).spawn(0), variant="scmoe")
    tokens = O.Rng(0).spawn(1).normal((T, d))
    cfg = SimpleNamespace(d_model=d, d_hidden=h, n_experts=N, variant="scmoe",
                          shortcut_pos="pos2", k_routed=1, combine_mode="direct_add",
                          capacity_factor=1.0, noise_enabled=False, pre_layernorm=False)
    blk = P.ScMoEBlockPair.from_reference(*_pair_ns(pp, cfg), dtype=torch.float32)
    out, dec, aux = blk(_t(tokens, torch.float32))
    idx = dec.indices.long().cpu().numpy()
    agree = (idx == z["idx"]).mean()
    assert agree > 0.99
    same = (idx[:, 0] == z["idx"][:, 0]) & (dec.dropped.cpu().numpy()[:, 0] == z["drop"][:, 0])
    o = out.double().cpu().numpy()
    # rows whose routing matches the reference reproduce its row sums
    ok, worst = O.allclose_scaled(o.sum(axis=1)[same], z["out_rowsum"][same], 1e-4)
    assert ok, worst
    _check(o[:16][same[:16]], z["out_head"][same[:16]], 1e-4, "cfg1 head rows")


@pytest.mark.parametrize("pos", ["pos1", "pos2", "pos3"])
def test_block_pair_slot_invariance_and_calibrate(pos):
    """Every expert slot gives bit-identical results; calibrate() picks a slot
    from measured costs."""
    T, d, h, N = 1024, 256, 1024, 8
    blk = P.ScMoEBlockPair(d, h, N, variant="scmoe", shortcut_pos=pos, n_heads=4, seq_len=256,
                           causal=True, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(0))
    x = torch.randn(T, d, device="cuda").bfloat16()
    outs = []
    for slot in range(len(P.sched.WINDOW_OPS[pos]) + 1):
        blk.slot = slot
        outs.append(blk(x)[0])
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    choice = blk.calibrate(x)
    assert 0 <= choice.slot <= len(P.sched.WINDOW_OPS[pos])


def test_full_size_cfg3_properties():
    """configs[2] shape (T=16384, d=2048, h=8192, N=8, cf=2): routing bit-exact
    on the kernel's logits, kept rows per expert <= quota, the routed output of
    a sample of tokens matches a torch reference of the same expert."""
    T, d, h, N = 16384, 2048, 8192, 8
    gen = torch.Generator(device="cuda").manual_seed(3)
    layer = P.ScMoELayer(d, h, N, capacity_factor=2.0, dtype=torch.bfloat16, generator=gen)
    x = torch.randn(T, d, device="cuda", generator=gen).bfloat16()
    src = torch.randn(T, d, device="cuda", generator=gen).bfloat16()
    out, dec, aux = layer(x, src)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    _check_routing(dec, dec.logits.double().cpu().numpy(), 1, 2.0)
    assert int(dec.kept_counts().max()) <= dec.quota
    se = layer.shared(x)
    sample = torch.arange(0, T, 97, device="cuda")
    e = dec.indices[sample, 0].long()
    for i, t in enumerate(sample.tolist()):
        if dec.dropped[t, 0]:
            expect = se[t].float()
        else:
            ei = int(e[i])
            hid = torch.nn.functional.gelu(src[t].float() @ layer.experts.w1t[ei].float().t()
                                           + layer.experts.b1[ei]).bfloat16()
            y = hid.float() @ layer.experts.w2t[ei].float().t() + layer.experts.b2[ei]
            expect = se[t].float() + y.bfloat16().float()
        err = (out[t].float() - expect).abs().max().item()
        assert err <= 2e-2 * (expect.abs().max().item() + 1e-3), (t, err)


def test_compat_shim_rebinds_moe_entries():
    """compat.install() swaps moe_shared / moe_standard of an arch-like module
    (here the oracle stands in for scmoelab.arch, which does not travel to the
    GPU box) and returns reference-shaped results."""
    from types import SimpleNamespace as NS
    from paper_2404_05019_b200 import compat

    class Decision:  # gating.GateDecision constructor signature
        def __init__(self, logits, indices, weights, dropped, eps=None):
            self.logits, self.indices, self.weights, self.dropped, self.eps = \
                logits, indices, weights, dropped, eps

    arch = NS(moe_shared=O.moe_shared, moe_standard=O.moe_standard)
    T, d, h, N, cf = 96, 32, 64, 4, 1.0
    pp = O.init_pair(d, h, N, O.Rng(8).spawn(0), variant="scmoe", combine_mode="cg2")
    x = O.Rng(8).spawn(1).normal((T, d))
    src = O.Rng(8).spawn(2).normal((T, d))
    compat.install(arch, dtype=torch.float32, gating_module=NS(GateDecision=Decision))
    try:
        cap = P.CapacityConfig(cf)
        out, dec, aux = arch.moe_shared(x, pp.moe, cap, 1, routed_src=src)
        assert isinstance(out, np.ndarray) and out.shape == (T, d) and aux.shape == (1, 1)
        ref, _, _ = O.moe_shared(x, pp.moe, cf, 1, routed_src=src, pinned_indices=dec.indices,
                                 pinned_dropped=dec.dropped)
        _check(out, ref, 1e-4, "compat moe_shared")
        pp2 = O.init_pair(d, h, N, O.Rng(9).spawn(0), variant="standard", k=2)
        out2, dec2, _ = arch.moe_standard(x, pp2.moe, cap, 2)
        ref2, _, _ = O.moe_standard(x, pp2.moe, cf, 2, pinned_indices=dec2.indices,
                                    pinned_dropped=dec2.dropped)
        _check(out2, ref2, 1e-4, "compat moe_standard")
    finally:
        compat.uninstall(arch)
    assert arch.moe_shared is O.moe_shared


def test_host_stream_runner_matches_direct_forward():
    from paper_2404_05019_b200.runtime import HostStreamRunner
    T, d, h, N = 512, 128, 256, 4
    blk = P.ScMoEBlockPair(d, h, N, variant="scmoe", shortcut_pos="pos2", n_heads=2, seq_len=128,
                           dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(4))
    xs = [torch.randn(T, d).bfloat16().pin_memory() for _ in range(5)]
    outs = [torch.empty(T, d, dtype=torch.bfloat16).pin_memory() for _ in range(5)]
    HostStreamRunner(lambda x: blk(x)).run(xs, outs)
    torch.cuda.synchronize()
    for x, o in zip(xs, outs):
        assert torch.equal(o, blk(x.cuda())[0].cpu())


@pytest.mark.parametrize("kw", [
    dict(n_blocks=4, variant="scmoe", shortcut_pos="pos2", first_layer_pos1=True),
    dict(n_blocks=3, variant="scmoe", shortcut_pos="pos1", moe_frequency="every-block"),
    dict(n_blocks=2, variant="standard", k_routed=2, moe_frequency="every-block"),
    dict(n_blocks=2, variant="shared", combine_mode="cg2", moe_frequency="every-block",
         pre_layernorm=True),
    dict(n_blocks=2, variant="scmoe", shortcut_pos="pos3", combine_mode="cg1")])
def test_model_matches_oracle_fp32(kw):
    """ScMoEModel (arch.model_forward on the GPU): pair stacks, first_layer_pos1,
    every-block placement, pre-LN — fp32 rtol 1e-4 with routing pinned."""
    T, d, h, N, cf = 256, 128, 256, 4, 1.0
    freq = kw.get("moe_frequency", "every-second-block")
    k = kw.get("k_routed", 1)
    blocks = O.init_model(kw["n_blocks"], d, h, N, O.Rng(21).spawn(0), moe_frequency=freq,
                          variant=kw["variant"], k=k, combine_mode=kw.get("combine_mode", "direct_add"))
    cfg = SimpleNamespace(n_blocks=kw["n_blocks"], d_model=d, d_hidden=h, n_experts=N, k_routed=k,
                          moe_frequency=freq, variant=kw["variant"],
                          shortcut_pos=kw.get("shortcut_pos"),
                          combine_mode=kw.get("combine_mode", "direct_add"), capacity_factor=cf,
                          noise_enabled=False, first_layer_pos1=kw.get("first_layer_pos1", False),
                          pre_layernorm=kw.get("pre_layernorm", False))
    model = P.ScMoEModel.from_reference(cfg, SimpleNamespace(blocks=blocks), dtype=torch.float32)
    tokens = O.Rng(21).spawn(1).normal((T, d))
    out, decs, auxes = model(_t(tokens, torch.float32))
    torch.cuda.synchronize()
    pinned = [(dd.indices.long().cpu().numpy(), dd.dropped.cpu().numpy()) for dd in decs]
    ref, rdecs, rauxes = O.model_forward(blocks, tokens, kw["variant"], kw.get("shortcut_pos"), cf,
                                         k, moe_frequency=freq,
                                         first_layer_pos1=kw.get("first_layer_pos1", False),
                                         pre_layernorm=kw.get("pre_layernorm", False),
                                         pinned=pinned)
    _check(out.double().cpu().numpy(), ref, 1e-4, f"model {kw}")
    for a, ra in zip(auxes, rauxes):
        assert float(a) == pytest.approx(ra, rel=1e-4, abs=1e-5)
    free = O.model_forward(blocks, tokens, kw["variant"], kw.get("shortcut_pos"), cf, k,
                           moe_frequency=freq, first_layer_pos1=kw.get("first_layer_pos1", False),
                           pre_layernorm=kw.get("pre_layernorm", False))[1]
    for dd, fd in zip(decs, free):
        assert (dd.indices.long().cpu().numpy() == fd.indices).mean() > 0.97


def test_every_block_training_step():
    """configs[3]-style every-block ScMoE (pos1) trains through the K7 kernels."""
    model = P.ScMoEModel(2, 128, 256, 4, moe_frequency="every-block", variant="scmoe",
                         shortcut_pos="pos1", n_heads=2, seq_len=128, capacity_factor=2.0,
                         dtype=torch.bfloat16,
                         generator=torch.Generator(device="cuda").manual_seed(3))
    model.requires_grad_(True)
    x = torch.randn(256, 128, device="cuda").bfloat16()
    tgt = torch.randn(256, 128, device="cuda").bfloat16()
    losses = [float(model.train_step(x, lr=2e-3, target=tgt)) for _ in range(6)]
    assert np.all(np.isfinite(losses)) and losses[-1] < losses[0]
    for blk in model.blocks:
        for p in (blk.attn_cur.w_qkv_t, blk.moe.experts.w1t, blk.moe.shared.b2, blk.moe.gate.w_gate_t):
            assert p.grad is not None and torch.isfinite(p.grad.float()).all()


@pytest.mark.parametrize("k,cf", [(1, 2.0), (1, 0.5), (2, 1.0)])
def test_fused_shared_combine_bit_identical(k, cf):
    """scmoe_shared_ffn_combine (combine in the SE GEMM2 epilogue) equals the
    shared expert followed by the combine kernel bit for bit (drops included)."""
    import paper_2404_05019_b200 as P
    from paper_2404_05019_b200 import kernels as K, layers as L
    T, d, h, N = 1000, 256, 512, 8
    layer = P.ScMoELayer(d, h, N, k_routed=k, capacity_factor=cf, dtype=torch.bfloat16,
                         generator=torch.Generator(device="cuda").manual_seed(4))
    x = torch.randn(T, d, device="cuda").bfloat16()
    src = torch.randn(T, d, device="cuda").bfloat16()
    res = torch.randn(T, d, device="cuda").bfloat16()
    with torch.no_grad():
        dec = layer.route(src)
        y = layer.routed_experts(src, dec)
        fused = layer.shared.forward_combine(x, y, dec, residual=res)
        se = layer.shared(x)
        ref = K.combine(y, dec.indices, dec.slots, dec.weights, dec.capacity, se_out=se,
                        residual=res)
        try:
            L.FUSED_COMBINE = False
            unfused_layer = layer(x, src, residual=res)[0]
        finally:
            L.FUSED_COMBINE = True
        fused_layer = layer(x, src, residual=res)[0]
    torch.cuda.synchronize()
    assert torch.equal(fused, ref)
    assert torch.equal(fused_layer, unfused_layer)


def _reference_package():
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ref = os.path.join(root, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "scmoelab")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from scmoelab import arch, gating, numkit
    return arch, gating, numkit


@pytest.mark.parametrize("variant,pos,mode,freq", [
    ("scmoe", "pos2", "cg1", "every-second-block"), ("scmoe", "pos1", "direct_add", "every-block"),
    ("standard", None, "direct_add", "every-second-block")])
def test_compat_drives_the_real_reference_model(variant, pos, mode, freq):
    """The unmodified reference (scmoelab, installed offline in baseline/_ref)
    runs its own arch.forward with compat.install() routing every MoE layer
    through our kernels; the result equals the reference's numpy forward
    replaying the GPU's routing decisions (fp32, rtol 1e-4)."""
    pkg = _reference_package()
    if pkg is None:
        pytest.skip("baseline/_ref (the installed reference) is not present")
    arch, gating, numkit = pkg
    from paper_2404_05019_b200 import compat
    n_blocks = 2 if freq == "every-second-block" else 3
    cfg = arch.ModelConfig(n_blocks=n_blocks, d_model=64, d_hidden=128, n_experts=4,
                           k_routed=1 if variant == "scmoe" else 2, moe_frequency=freq,
                           variant=variant, shortcut_pos=pos, combine_mode=mode,
                           capacity_factor=1.0)
    params = arch.init_params(cfg, numkit.Rng(3))
    tokens = numkit.Rng(4).normal((96, 64))
    compat.install(dtype=torch.float32)
    try:
        gpu_out, gpu_trace = arch.forward(cfg, params, tokens)
    finally:
        compat.uninstall()
    assert arch.moe_shared.__module__.startswith("scmoelab")
    ref_out, _ = arch.forward(cfg, params, tokens, replay=arch.replay_from_trace(gpu_trace))
    _check(gpu_out, ref_out, 1e-4, "reference arch.forward through compat")


@pytest.mark.parametrize("pos", ["pos1", "pos2", "pos3"])
def test_routed_side_stream_bit_identical(pos):
    """Inference with the routed ops on the side stream (routed_stream_infer,
    the default) equals the serial issue order bit for bit, eager and inside a
    CUDA graph, with the fused shared-expert combine."""
    from paper_2404_05019_b200.runtime import CapturedStep
    T, d, h, N = 2048, 256, 512, 8
    blk = P.ScMoEBlockPair(d, h, N, variant="scmoe", shortcut_pos=pos, n_heads=4, seq_len=256,
                           causal=True, capacity_factor=1.25, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(31))
    x = torch.randn(T, d, device="cuda", generator=torch.Generator(device="cuda").manual_seed(32))
    x = x.bfloat16()
    with torch.no_grad():
        blk.routed_stream_infer = False
        ref, dref, _ = blk(x)
        ref = ref.clone()
        for mode in (True, "decode"):        # join in the shared expert / at the combine
            blk.routed_stream_infer = mode
            out, dec, _ = blk(x)
            torch.cuda.synchronize()
            assert torch.equal(out, ref), mode
            assert torch.equal(dec.slots, dref.slots) and torch.equal(dec.indices, dref.indices)
            g = CapturedStep(lambda xx: blk(xx)[0], [x])
            assert torch.equal(g.replay().clone(), ref), mode


def test_every_block_routed_side_stream_bit_identical():
    """The every-block placement (ScMoEBlock, pos1) with the routed ops on the
    side stream equals the serial order bit for bit."""
    T, d, h, N = 1024, 256, 512, 16
    blk = P.ScMoEBlock(d, h, N, variant="scmoe", shortcut_pos="pos1", n_heads=4, seq_len=256,
                       causal=True, capacity_factor=2.0, dtype=torch.bfloat16,
                       generator=torch.Generator(device="cuda").manual_seed(41))
    x = torch.randn(T, d, device="cuda", generator=torch.Generator(device="cuda").manual_seed(42))
    x = x.bfloat16()
    with torch.no_grad():
        blk.routed_stream_infer = False
        ref = blk(x)[0].clone()
        blk.routed_stream_infer = "decode"
        out = blk(x)[0]
        torch.cuda.synchronize()
    assert torch.equal(out, ref)
