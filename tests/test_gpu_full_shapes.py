"""Parity at the BASELINE.json shapes themselves (not scaled-down stand-ins).

The checker is an independent torch fp32 computation of arch.moe_shared
(arch.py:496-504) from the layer's own bf16 weights, on a sample of tokens:
  SE(x)   = gelu(x W1 + b1) W2 + b2        (expert_forward, arch.py:349-351,
            exact erf GELU; the hidden row rounded to bf16 as the kernels
            store it)
  routed  = Y_e(src) for the token's kept expert, 0 when dropped
  out     = SE(x) + routed (+ residual)    (direct add, arch.py:380-392, 616)
with the GPU's routing (bit-exact on its own logits, checked separately).
None of the product's kernels is used to build the expectation.
Tolerance: bf16, |gpu - ref| <= 2e-2 (|ref| + max|ref|) (north star rtol
2e-2 with the scaled atol of SURVEY §7)."""

import numpy as np
import pytest
import torch

from oracle import scmoe_oracle as O

pytestmark = pytest.mark.gpu
P = None
RTOL = 2e-2


def setup_module(module):
    global P
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2404_05019_b200 as pkg
    P = pkg


def _ffn_ref(x, w1t, b1, w2t, b2):
    """fp32 expert_forward from bf16 weights; hidden rounded to bf16."""
    hid = torch.nn.functional.gelu(x.float() @ w1t.float().t() + b1.float())
    return hid.bfloat16().float() @ w2t.float().t() + b2.float()


def _layer_ref(layer, x_cur, src, dec, sample, residual=None):
    torch.backends.cuda.matmul.allow_tf32 = False
    sh = layer.shared
    exp = _ffn_ref(x_cur[sample], sh.w1t, sh.b1, sh.w2t, sh.b2).bfloat16().float()
    e = dec.indices[sample, 0].long()
    kept = ~dec.dropped[sample, 0]
    routed = torch.zeros_like(exp)
    ex = layer.experts
    for ei in range(ex.n_experts):
        m = (e == ei) & kept
        if bool(m.any()):
            rows = sample[m]
            routed[m] = _ffn_ref(src[rows], ex.w1t[ei], ex.b1[ei], ex.w2t[ei],
                                 ex.b2[ei]).bfloat16().float()
    out = exp + routed
    if residual is not None:
        out = out + residual[sample].float()
    return out


def _check(gpu, ref, what):
    ok, worst = O.allclose_scaled(gpu.double().cpu().numpy(), ref.double().cpu().numpy(), RTOL)
    assert ok, f"{what}: worst error / bound = {worst:.3g}"


def _routing_exact(dec, k, cf):
    lg = dec.logits.double().cpu().numpy()
    ref = O.apply_capacity(O.select_topk(lg, k), cf, lg.shape[1], lg.shape[0])
    np.testing.assert_array_equal(dec.indices.long().cpu().numpy(), ref.indices)
    np.testing.assert_array_equal(dec.dropped.cpu().numpy(), ref.dropped)


def test_configs2_layer_full_tokens_fused_combine():
    """configs[2]: T = 16384, d 2048, h 8192, N 8, cf 2.0 — the inference
    default (the combine fused into the shared expert's GEMM2 epilogue, with
    the block residual) on 4096 sampled tokens (every 4th), plus the unfused
    path bit-identical on ALL tokens."""
    T, d, h, N, cf = 16384, 2048, 8192, 8, 2.0
    gen = torch.Generator(device="cuda").manual_seed(21)
    layer = P.ScMoELayer(d, h, N, capacity_factor=cf, dtype=torch.bfloat16, generator=gen)
    x = torch.randn(T, d, device="cuda", generator=gen).bfloat16()
    src = torch.randn(T, d, device="cuda", generator=gen).bfloat16()
    res = torch.randn(T, d, device="cuda", generator=gen).bfloat16()
    with torch.no_grad():
        out, dec, _ = layer(x, src, residual=res)
        torch.cuda.synchronize()
        assert layer.shared.can_fuse_combine(x, dec, layer.combine_mode)
        _routing_exact(dec, 1, cf)
        assert int(dec.kept_counts().max()) <= dec.quota
        sample = torch.arange(0, T, 4, device="cuda")
        _check(out[sample], _layer_ref(layer, x, src, dec, sample, residual=res),
               "configs[2] fused layer")
        # the fused epilogue equals the separate SE GEMM + combine kernel bit
        # for bit, on every token
        try:
            P.layers.FUSED_COMBINE = False
            out2, _, _ = layer(x, src, residual=res)
        finally:
            P.layers.FUSED_COMBINE = True
        torch.cuda.synchronize()
        assert torch.equal(out, out2)


def test_configs2_block_pair_full_tokens():
    """The configs[2] block pair (32 heads, causal 2048-token sequences x 8):
    the MoE feed of the block's own x_cur / src taps vs the fp32 reference on
    2048 sampled tokens, residual included (out = h_mh_cur + feed)."""
    T, d, h, N = 16384, 2048, 8192, 8
    blk = P.ScMoEBlockPair(d, h, N, variant="scmoe", shortcut_pos="pos2", n_heads=32,
                           seq_len=2048, causal=True, capacity_factor=2.0, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(22))
    x = torch.randn(T, d, device="cuda").bfloat16()
    with torch.no_grad():
        out, dec, _, taps = blk(x, return_taps=True)
        torch.cuda.synchronize()
        sample = torch.arange(3, T, 8, device="cuda")
        ref = _layer_ref(blk.moe, taps["x_cur"], taps["src"], dec, sample,
                         residual=taps["h_mh_cur"])
        _check(out[sample], ref, "configs[2] block pair")


def test_configs3_every_block_full_shape():
    """configs[3]: every-block placement, pos1, d 4096, h 16384, N 16 (all
    16 experts on this GPU), 4 causal 2048-token sequences = 8192 tokens:
    routing bit-exact, the MoE feed vs the fp32 reference on 1024 sampled
    tokens (GEMMs at K = 4096 -> 16384 and 16384 -> 4096, 16 groups)."""
    T, d, h, N, cf = 8192, 4096, 16384, 16, 2.0
    blk = P.ScMoEBlock(d, h, N, variant="scmoe", shortcut_pos="pos1", n_heads=32, seq_len=2048,
                       causal=True, capacity_factor=cf, dtype=torch.bfloat16,
                       generator=torch.Generator(device="cuda").manual_seed(23))
    x = torch.randn(T, d, device="cuda").bfloat16()
    with torch.no_grad():
        out, dec, _, taps = blk(x, return_taps=True)
        torch.cuda.synchronize()
        assert torch.equal(taps["src"], x)            # pos1 every-block: src = h_in
        _routing_exact(dec, 1, cf)
        assert int(dec.counts.gt(0).sum()) == N       # all 16 experts routed to
        sample = torch.arange(5, T, 8, device="cuda")
        ref = _layer_ref(blk.moe, taps["x_cur"], taps["src"], dec, sample,
                         residual=taps["h_mh_cur"])
        _check(out[sample], ref, "configs[3] every-block")


def test_configs3_attention_projection_gemm():
    """The every-block attention projections at configs[3] width (QKV 4096 ->
    12288, O 4096 -> 4096 + residual) vs fp32 torch on 512 rows."""
    from paper_2404_05019_b200 import kernels as K
    torch.backends.cuda.matmul.allow_tf32 = False
    T, d = 8192, 4096
    g = torch.Generator(device="cuda").manual_seed(24)
    x = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    wqkv = (torch.randn(3 * d, d, device="cuda", generator=g) / 64).bfloat16()
    wo = (torch.randn(d, d, device="cuda", generator=g) / 64).bfloat16()
    res = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    qkv = K.grouped_gemm(x, wqkv, None)
    o = K.grouped_gemm(x, wo, None, residual=res)
    rows = torch.arange(7, T, 16, device="cuda")
    _check(qkv[rows], x[rows].float() @ wqkv.float().t(), "qkv 4096->12288")
    _check(o[rows], x[rows].float() @ wo.float().t() + res[rows].float(), "o 4096->4096 + res")
