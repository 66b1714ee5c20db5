"""Training step (K7) parity: gradients of the reference objective
(loss + 0.01 * aux, grad.py:52-67) from the bf16 GPU backward vs the float64
gradient oracle (oracle/grad_oracle.py, itself pinned to the reference's tape
gradients), at the same bf16-rounded parameters and inputs, with the GPU's
routing pinned (straight-through, tape.py:11-13).

Tolerance: |g_gpu - g_ref| <= rtol * (|g_ref| + max|g_ref|) per parameter
tensor with rtol = 5e-2 — the bf16 backward stacks several bf16 roundings of
activations and gradients on top of the forward's 2e-2 budget.
"""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import grad_oracle as G
from oracle import scmoe_oracle as O

pytestmark = pytest.mark.gpu
P = None
RTOL = 5e-2


def setup_module(module):
    global P
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2404_05019_b200 as pkg
    P = pkg


def _expert_items(prefix, w1t, b1, w2t, b2):
    return {prefix + ".w1": w1t.t(), prefix + ".b1": b1.reshape(1, -1),
            prefix + ".w2": w2t.t(), prefix + ".b2": b2.reshape(1, -1)}


def _ref_view(blk, grad=False):
    """Module tensors (or their .grad) under the reference's names/shapes."""
    g = (lambda t: t.grad) if grad else (lambda t: t.detach())
    d = blk.attn_prev.d_model
    out = {}
    for bi, att in ((0, blk.attn_prev), (1, blk.attn_cur)):
        qkv = g(att.w_qkv_t)
        for j, nm in enumerate(("w_q", "w_k", "w_v")):
            out[f"block{bi}.attn.{nm}"] = qkv[j * d:(j + 1) * d].t()
        out[f"block{bi}.attn.w_o"] = g(att.w_o_t).t()
    m = blk.mlp_prev
    out.update(_expert_items("block0.mlp", g(m.w1t), g(m.b1), g(m.w2t), g(m.b2)))
    moe = blk.moe
    e = moe.experts
    for i in range(e.n_experts):
        out.update(_expert_items(f"block1.moe.expert{i}", g(e.w1t)[i], g(e.b1)[i], g(e.w2t)[i],
                                 g(e.b2)[i]))
    if hasattr(moe, "shared"):
        s = moe.shared
        out.update(_expert_items("block1.moe.shared", g(s.w1t), g(s.b1), g(s.w2t), g(s.b2)))
        if moe.w_cg is not None:
            out["block1.moe.cg.w"] = g(moe.w_cg)
    out["block1.moe.gate.w_gate"] = g(moe.gate.w_gate_t).t()
    wn = g(moe.gate.w_noise_t)
    out["block1.moe.gate.w_noise"] = (wn if wn is not None
                                      else torch.zeros_like(moe.gate.w_noise_t)).t()
    return {k: v.double().cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("variant,pos,mode,k,cf,mse", [
    ("scmoe", "pos2", "direct_add", 1, 1.0, False), ("scmoe", "pos1", "cg1", 1, 2.0, True),
    ("scmoe", "pos3", "cg2", 1, 0.75, False), ("standard", None, "direct_add", 2, 1.0, True),
    ("shared", None, "direct_add", 2, 2.0, False)])
def test_block_pair_gradients(variant, pos, mode, k, cf, mse):
    T, d, h, N = 256, 128, 256, 4
    pp = O.init_pair(d, h, N, O.Rng(17).spawn(0), variant=variant, k=k, combine_mode=mode)
    cfg = SimpleNamespace(d_model=d, d_hidden=h, n_experts=N, variant=variant, shortcut_pos=pos,
                          k_routed=k, combine_mode=mode, capacity_factor=cf, noise_enabled=False,
                          pre_layernorm=False)
    prev = SimpleNamespace(attn=pp.attn_prev, feed=pp.mlp_prev)
    cur = SimpleNamespace(attn=pp.attn_cur, feed=pp.moe)
    blk = P.ScMoEBlockPair.from_reference(cfg, prev, cur, dtype=torch.bfloat16)
    with torch.no_grad():                       # non-zero biases exercise the bias grads
        for prm in (blk.mlp_prev.b1, blk.moe.experts.b2):
            prm.copy_(torch.randn_like(prm) * 0.1)
    blk.requires_grad_(True)
    x = torch.as_tensor(O.Rng(17).spawn(1).normal((T, d)), device="cuda").bfloat16()
    target = torch.randn(T, d, device="cuda").bfloat16() if mse else None
    params0 = _ref_view(blk)                    # bf16-rounded parameters, float64
    out, dec, aux = blk(x)
    loss = (out.float().mean() if target is None
            else (out.float() - target.float()).pow(2).sum() / T) + 0.01 * aux
    loss.backward()
    torch.cuda.synchronize()
    ref_loss, ref_grads = G.pair_grads(
        params0, x.double().cpu().numpy(), variant=variant, pos=pos, n_experts=N, k=k,
        combine_mode=mode, pinned_indices=dec.indices.long().cpu().numpy(),
        pinned_dropped=dec.dropped.cpu().numpy(),
        target=None if target is None else target.double().cpu())
    assert float(loss) == pytest.approx(ref_loss, rel=2e-2, abs=1e-3)
    got = _ref_view(blk, grad=True)
    for name, ref in ref_grads.items():
        if name not in got:
            continue
        gv = got[name]
        bound = RTOL * (np.abs(ref) + np.abs(ref).max() + 1e-30)
        worst = float((np.abs(gv - ref) / bound).max())
        assert worst <= 1.0, f"{variant}/{mode} grad {name}: worst err/bound {worst:.3g}"


def test_train_step_reduces_loss_and_updates():
    """A few SGD steps of the reference objective on a fixed target lower the
    loss (the reference's toy trainer, grad.py:296-333)."""
    T, d, h, N = 512, 128, 256, 4
    blk = P.ScMoEBlockPair(d, h, N, variant="scmoe", shortcut_pos="pos2", n_heads=2, seq_len=128,
                           capacity_factor=1.25, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(5))
    blk.requires_grad_(True)
    g = torch.Generator(device="cuda").manual_seed(6)
    x = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    target = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    w_before = blk.moe.experts.w1t.detach().clone()
    losses = [float(blk.train_step(x, lr=2e-3, target=target)) for _ in range(8)]
    assert losses[-1] < losses[0]
    assert not torch.equal(w_before, blk.moe.experts.w1t.detach())
    assert all(np.isfinite(losses))


def test_train_step_nonfinite_loss_raises_before_update():
    """check_finite: a non-finite loss raises FloatingPointError and leaves the
    parameters untouched (grad.py:84-85, 322-323)."""
    T, d, h, N = 256, 128, 256, 4
    blk = P.ScMoEBlockPair(d, h, N, variant="scmoe", shortcut_pos="pos2", n_heads=2, seq_len=128,
                           capacity_factor=1.25, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(7))
    blk.requires_grad_(True)
    x = torch.randn(T, d, device="cuda").bfloat16()
    target = torch.full((T, d), float("inf"), device="cuda").bfloat16()
    w_before = blk.moe.experts.w1t.detach().clone()
    with pytest.raises(FloatingPointError, match="non-finite loss"):
        blk.train_step(x, lr=1e-3, target=target, check_finite=True)
    assert torch.equal(w_before, blk.moe.experts.w1t.detach())
    assert torch.isfinite(blk.train_step(x, lr=1e-3, check_finite=True)).item()


def _check_grads(got, ref_grads, tag):
    for name, ref in ref_grads.items():
        if name not in got:
            continue
        gv = got[name]
        bound = RTOL * (np.abs(ref) + np.abs(ref).max() + 1e-30)
        worst = float((np.abs(gv - ref) / bound).max())
        assert worst <= 1.0, f"{tag} grad {name}: worst err/bound {worst:.3g}"


@pytest.mark.parametrize("variant,k", [("scmoe", 1), ("standard", 2)])
def test_noisy_gate_gradients(variant, k):
    """Training with the noisy gate (arch.py:405-415): the logits carry
    eps * softplus(src W_noise) and the gate's backward differentiates through
    it — W_gate, W_noise and the source rows get the reference tape's
    gradients (recorded draws pinned, MoEReplay semantics)."""
    T, d, h, N = 256, 128, 256, 6
    pp = O.init_pair(d, h, N, O.Rng(23).spawn(0), variant=variant, k=k, noise_enabled=True)
    cfg = SimpleNamespace(d_model=d, d_hidden=h, n_experts=N, variant=variant,
                          shortcut_pos="pos2" if variant == "scmoe" else None, k_routed=k,
                          combine_mode="direct_add", capacity_factor=1.0, noise_enabled=True,
                          pre_layernorm=False)
    blk = P.ScMoEBlockPair.from_reference(cfg, SimpleNamespace(attn=pp.attn_prev, feed=pp.mlp_prev),
                                          SimpleNamespace(attn=pp.attn_cur, feed=pp.moe),
                                          dtype=torch.bfloat16)
    blk.requires_grad_(True)
    x = torch.as_tensor(O.Rng(23).spawn(1).normal((T, d)), device="cuda").bfloat16()
    eps = torch.as_tensor(O.Rng(23).spawn(2).normal((T, N)), device="cuda").float()
    params0 = _ref_view(blk)
    out, dec, aux = blk(x, eps=eps)
    loss = out.float().mean() + 0.01 * aux
    loss.backward()
    torch.cuda.synchronize()
    assert dec.eps is not None
    ref_loss, ref_grads = G.pair_grads(
        params0, x.double().cpu().numpy(), variant=variant, pos=cfg.shortcut_pos, n_experts=N,
        k=k, combine_mode="direct_add", pinned_indices=dec.indices.long().cpu().numpy(),
        pinned_dropped=dec.dropped.cpu().numpy(), eps=eps.double().cpu().numpy())
    assert float(loss) == pytest.approx(ref_loss, rel=2e-2, abs=1e-3)
    got = _ref_view(blk, grad=True)
    assert np.abs(got["block1.moe.gate.w_noise"]).max() > 0
    _check_grads(got, ref_grads, f"noisy {variant}")


def test_configs1_shape_gradients():
    """configs[1] at its real widths (SwinV2-MoE-S stage 3: d 384, h 1536, 12
    heads over 12x12 = 144-token windows, cf 1.25) with 8 experts, on a
    1152-token subsample (8 windows): every parameter's gradient vs the
    float64 oracle."""
    T, d, h, N, heads, S = 1152, 384, 1536, 8, 12, 144
    pp = O.init_pair(d, h, N, O.Rng(29).spawn(0), variant="scmoe")
    cfg = SimpleNamespace(d_model=d, d_hidden=h, n_experts=N, variant="scmoe",
                          shortcut_pos="pos2", k_routed=1, combine_mode="direct_add",
                          capacity_factor=1.25, noise_enabled=False, pre_layernorm=False)
    blk = P.ScMoEBlockPair.from_reference(cfg, SimpleNamespace(attn=pp.attn_prev, feed=pp.mlp_prev),
                                          SimpleNamespace(attn=pp.attn_cur, feed=pp.moe),
                                          dtype=torch.bfloat16, n_heads=heads, seq_len=S)
    blk.requires_grad_(True)
    x = torch.as_tensor(O.Rng(29).spawn(1).normal((T, d)), device="cuda").bfloat16()
    params0 = _ref_view(blk)
    out, dec, aux = blk(x)
    loss = out.float().mean() + 0.01 * aux
    loss.backward()
    torch.cuda.synchronize()
    assert int(dec.counts.gt(0).sum()) == N     # every expert gets rows (and gradients)
    ref_loss, ref_grads = G.pair_grads(
        params0, x.double().cpu().numpy(), variant="scmoe", pos="pos2", n_experts=N, k=1,
        combine_mode="direct_add", pinned_indices=dec.indices.long().cpu().numpy(),
        pinned_dropped=dec.dropped.cpu().numpy(), n_heads=heads, seq_len=S)
    assert float(loss) == pytest.approx(ref_loss, rel=2e-2, abs=1e-3)
    _check_grads(_ref_view(blk, grad=True), ref_grads, "configs[1]")


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("N,k,noise", [(8, 1, False), (8, 2, True), (12, 2, False),
                                       (40, 3, True)])
def test_gate_backward_kernel(dtype, N, k, noise):
    """scmoe_gate_backward vs float64 autograd of the same objective:
    d(c_aux * aux + <dw, weights>) through H = src Wg (+ eps softplus(src Wn))."""
    from paper_2404_05019_b200 import kernels as K
    T, d = 1001, 256
    g = torch.Generator(device="cuda").manual_seed(N * 10 + k)
    src = torch.randn(T, d, device="cuda", generator=g).to(dtype)
    wg = torch.randn(N, d, device="cuda", generator=g) / 16
    wn = torch.randn(N, d, device="cuda", generator=g) / 16
    eps = torch.randn(T, N, device="cuda", generator=g)
    logits = src.float() @ wg.t()
    noise_pre = src.float() @ wn.t()
    if noise:
        logits = logits + eps * torch.nn.functional.softplus(noise_pre)
    idx = torch.topk(logits, k, dim=1).indices.to(torch.int32)
    w = torch.softmax(logits.gather(1, idx.long()), dim=1)
    counts = torch.bincount(idx.reshape(-1).long(), minlength=N).to(torch.int32)
    dw = torch.randn(T, k, device="cuda", generator=g)
    d_aux = torch.tensor(0.37, device="cuda")
    d_src, d_wg, d_wn = K.gate_backward(
        src, logits.contiguous(), idx, w.contiguous(), counts, wg, d_weights=dw, d_aux=d_aux,
        w_noise_t=wn if noise else None, eps=eps if noise else None,
        noise_pre=noise_pre.contiguous() if noise else None)
    # float64 autograd reference
    s64 = src.double().requires_grad_(True)
    g64 = wg.double().requires_grad_(True)
    n64 = wn.double().requires_grad_(True)
    h = s64 @ g64.t()
    if noise:
        h = h + eps.double() * torch.nn.functional.softplus(s64 @ n64.t())
    sel = h.gather(1, idx.long())
    wsel = torch.softmax(sel, dim=1)
    f = counts.double() / (T * k)
    aux = N * (torch.softmax(h, dim=1).mean(0) * f).sum()
    obj = 0.37 * aux + ((wsel * dw.double()).sum() if k > 1 else 0.0)
    obj.backward()
    def close(a, b, tol):
        b = b.detach()
        err = (a.double() - b).abs().max().item()
        assert err <= tol * (b.abs().max().item() + 1e-12), (err, b.abs().max().item())
    tol = 1e-2 if dtype == torch.bfloat16 else 1e-4
    close(d_src, s64.grad, tol)
    close(d_wg, g64.grad, 1e-4)
    if noise:
        close(d_wn, n64.grad, 1e-4)


@pytest.mark.parametrize("n_exp", [1, 8])
def test_concurrent_backward_matches_serial(n_exp):
    """training.CONCURRENT_BWD (weight gradients on a side stream, half of the
    SMs per GEMM) gives the serial backward's gradients: same kernels, only
    the split-K split count of the weight gradients changes with the SM
    budget (fp32 partials, a different summation order), inside a CUDA graph
    too (the side stream forks from and joins the capture stream)."""
    from paper_2404_05019_b200 import training as TR
    from paper_2404_05019_b200.runtime import CapturedStep
    T, d, h = 2304, 384, 1536
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    grads = {}
    old = TR.CONCURRENT_BWD
    try:
        for conc in (False, True):
            TR.CONCURRENT_BWD = conc
            blk = P.ScMoEBlockPair(d, h, n_exp, variant="scmoe", shortcut_pos="pos2", n_heads=12,
                                   seq_len=144, capacity_factor=1.25, dtype=torch.bfloat16,
                                   generator=torch.Generator(device="cuda").manual_seed(12))
            blk.requires_grad_(True)
            step = CapturedStep(lambda xx, b=blk: b.train_step(xx, lr=0.0), [x], warmup=1)
            step.replay()
            torch.cuda.synchronize()
            grads[conc] = {n: p.grad.detach().float().clone()
                           for n, p in blk.named_parameters() if p.grad is not None}
    finally:
        TR.CONCURRENT_BWD = old
    assert grads[False].keys() == grads[True].keys() and len(grads[True]) > 10
    for n in grads[True]:
        a, b = grads[False][n], grads[True][n]
        scale = a.abs().max().clamp_min(1e-6)
        assert float((a - b).abs().max() / scale) < 2e-2, n
