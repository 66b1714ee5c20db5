"""Windowed attention kernels (csrc/attention.cu) vs torch fp32 attention on
the same bf16 inputs: forward output, the row log-sum-exp, and the backward's
packed dQKV.  Semantics: per window and head O = softmax(Q K^T scale) V
(arch.py:354-358 generalised to heads / windows / causal masking).
Tolerance: |gpu - ref| <= rtol (|ref| + max|ref|), rtol 2e-2 forward (bf16
P and O), 3e-2 backward (bf16 dS)."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu
K = None


def setup_module(module):
    global K
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_05019_b200 import kernels
    K = kernels


def _close(a, b, rtol, what):
    a, b = a.double(), b.double()
    bound = rtol * (b.abs() + b.abs().max())
    worst = float(((a - b).abs() / bound).max())
    assert worst <= 1.0, f"{what}: worst err/bound {worst:.3g}"


def _ref(qkv, H, S, scale, causal):
    T, d3 = qkv.shape
    d = d3 // 3
    hd = d // H
    q, k, v = qkv.float().view(T // S, S, 3, H, hd).permute(2, 0, 3, 1, 4).unbind(0)
    s = (q @ k.transpose(-1, -2)) * scale
    if causal:
        s = s.masked_fill(torch.ones(S, S, dtype=torch.bool, device=s.device).triu(1),
                          float("-inf"))
    lse = torch.logsumexp(s, dim=-1) / math.log(2.0)            # base 2
    o = torch.softmax(s, dim=-1) @ v
    return o.permute(0, 2, 1, 3).reshape(T, d), lse.permute(0, 2, 1).reshape(T, H)


@pytest.mark.parametrize("S,H,hd,causal", [(144, 12, 32, False), (144, 3, 64, False),
                                           (64, 4, 64, True), (192, 2, 32, False),
                                           (16, 5, 32, True), (128, 8, 32, True)])
def test_window_attention_fwd_bwd(S, H, hd, causal):
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device="cuda").manual_seed(S + H + hd)
    nw = 6
    T, d = nw * S, H * hd
    qkv = torch.randn(T, 3 * d, device="cuda", generator=g).bfloat16()
    scale = 1.0 / math.sqrt(hd)
    o, lse = K.window_attention_fwd(qkv, H, S, scale, causal)
    ref_o, ref_lse = _ref(qkv, H, S, scale, causal)
    _close(o, ref_o, 2e-2, "O")
    _close(lse, ref_lse, 1e-3, "lse")
    # backward vs fp32 autograd
    dout = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    dqkv = K.window_attention_bwd(qkv, o, dout, lse, H, S, scale, causal)
    x = qkv.float().requires_grad_(True)
    ro, _ = _ref(x, H, S, scale, causal)
    ro.backward(dout.float())
    for i, nm in enumerate(("dQ", "dK", "dV")):
        _close(dqkv[:, i * d:(i + 1) * d], x.grad[:, i * d:(i + 1) * d], 3e-2, nm)


def test_attention_module_window_vs_library():
    """block.Attention training step on the window kernels equals the
    library (cuDNN SDPA) path within bf16 tolerance: output and every
    gradient."""
    import paper_2404_05019_b200 as P
    from paper_2404_05019_b200 import block
    T, d, H, S = 144 * 8, 384, 12, 144
    outs, grads = [], []
    for use in (True, False):
        block.WINDOW_ATTENTION = use
        try:
            att = P.Attention(d, H, S, causal=False, dtype=torch.bfloat16,
                              generator=torch.Generator(device="cuda").manual_seed(3))
            att.requires_grad_(True)
            x = torch.randn(T, d, device="cuda",
                            generator=torch.Generator(device="cuda").manual_seed(4)).bfloat16()
            x.requires_grad_(True)
            y = att(x, residual=x)
            y.float().square().mean().backward()
            outs.append(y.detach())
            grads.append([x.grad, att.w_qkv_t.grad, att.w_o_t.grad])
        finally:
            block.WINDOW_ATTENTION = True
    _close(outs[0], outs[1], 2e-2, "out")
    for a, b, nm in zip(grads[0], grads[1], ("dx", "dWqkv", "dWo")):
        _close(a, b, 3e-2, nm)
