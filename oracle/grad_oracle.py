"""Gradient oracle — TEST INFRASTRUCTURE ONLY.

A float64 restatement, on torch autograd, of the reference's training
objective for one block pair: `grad.compute_loss` (grad.py:52-67) over
`arch.model_forward`'s pair loop (arch.py:580-631) with the tape semantics
of tape.py (straight-through routing: index sets and drop masks are
constants, tape.py:11-13; masked-softmax weights, tape.py:161-176; exact-erf
GELU, tape.py:137-142; balance loss through the full softmax,
arch.py:436-439, 484-485).

It is pinned against gradients the reference itself produced
(`grad.backward`, golden vectors in tests/golden/grad_cases.npz) by
tests/test_oracle_golden.py, and used by the GPU tests as the checker for the
bf16 backward kernels.  The product never imports it.

Parameters use the reference's names (`arch.named_parameters`,
arch.py:204-224) with the reference's shapes: w1 (d, h), b1 (1, h), ...
"""

from __future__ import annotations

import math
from typing import Dict, Optional

import numpy as np
import torch


def _gelu(x):
    return 0.5 * x * (1.0 + torch.erf(x / math.sqrt(2.0)))


def _expert(x, p, prefix):
    return _gelu(x @ p[prefix + ".w1"] + p[prefix + ".b1"]) @ p[prefix + ".w2"] + p[prefix + ".b2"]


def _attention(x, p, prefix, d_model, n_heads=1, seq_len=None, causal=False):
    """Single-head unmasked SDPA with 1/sqrt(d_model) scale (arch.py:354-358);
    n_heads > 1 / seq_len / causal generalise it the way block.Attention does."""
    q, k, v = x @ p[prefix + ".w_q"], x @ p[prefix + ".w_k"], x @ p[prefix + ".w_v"]
    t = x.shape[0]
    s = seq_len or t
    hd = d_model // n_heads
    scale = 1.0 / math.sqrt(d_model) if n_heads == 1 else 1.0 / math.sqrt(hd)

    def split(z):
        return z.view(t // s, s, n_heads, hd).permute(0, 2, 1, 3)

    qh, kh, vh = split(q), split(k), split(v)
    sc = (qh @ kh.transpose(-1, -2)) * scale
    if causal:
        mask = torch.ones(s, s, dtype=torch.bool, device=x.device).triu(1)
        sc = sc.masked_fill(mask, float("-inf"))
    o = torch.softmax(sc, dim=-1) @ vh
    o = o.permute(0, 2, 1, 3).reshape(t, d_model)
    return o @ p[prefix + ".w_o"]


def pair_loss(p: Dict[str, torch.Tensor], tokens: torch.Tensor, variant: str, pos: Optional[str],
              n_experts: int, k: int, combine_mode: str, pinned_indices, pinned_dropped,
              aux_coeff: float = 0.01, target: Optional[torch.Tensor] = None,
              n_heads: int = 1, seq_len: Optional[int] = None, causal: bool = False,
              eps=None):
    """Loss of one block pair (blocks 0 and 1) with routing pinned; returns
    (loss, out).  eps (T, N): the noisy gate's recorded draws, H = src W_gate
    + eps * softplus(src W_noise) (arch.py:405-415), differentiated through
    (tape.py: mm, mul, softplus)."""
    d = tokens.shape[1]
    h_in = tokens
    h_mh_prev = h_in + _attention(h_in, p, "block0.attn", d, n_heads, seq_len, causal)
    h_mlp_prev = h_mh_prev + _expert(h_mh_prev, p, "block0.mlp")
    h_mh_cur = h_mlp_prev + _attention(h_mlp_prev, p, "block1.attn", d, n_heads, seq_len, causal)
    x_cur = h_mh_cur
    if variant == "scmoe":
        src = {"pos1": h_mlp_prev, "pos2": h_mh_prev, "pos3": h_in}[pos]
    else:
        src = x_cur
    logits = src @ p["block1.moe.gate.w_gate"]
    if eps is not None:
        e = torch.as_tensor(np.asarray(eps), dtype=logits.dtype, device=logits.device)
        logits = logits + e * torch.nn.functional.softplus(src @ p["block1.moe.gate.w_noise"])
    t = logits.shape[0]
    idx = torch.as_tensor(np.asarray(pinned_indices), dtype=torch.long, device=logits.device)
    drop = torch.as_tensor(np.asarray(pinned_dropped), dtype=torch.bool, device=logits.device)
    support = torch.zeros_like(logits, dtype=torch.bool).scatter(1, idx, True)
    keep = torch.zeros_like(logits).scatter(1, idx, (~drop).to(logits.dtype))
    probs = torch.softmax(logits.masked_fill(~support, float("-inf")), dim=1)
    wmat = probs * keep                                           # arch.py:481-482
    routed = torch.zeros_like(src)
    for i in range(n_experts):                                    # arch.py:418-433
        if bool((keep[:, i] != 0).any()):
            routed = routed + wmat[:, i:i + 1] * _expert(src, p, f"block1.moe.expert{i}")
    counts = torch.bincount(idx.reshape(-1), minlength=n_experts).to(logits.dtype)
    f = counts / float(t * k)
    aux = n_experts * (torch.softmax(logits, dim=1).mean(0) * f).sum()   # arch.py:436-439
    if variant == "standard":
        feed = routed
    else:
        se = _expert(x_cur, p, "block1.moe.shared")
        if combine_mode == "direct_add":
            feed = se + routed
        else:
            z = x_cur @ p["block1.moe.cg.w"].t()
            if combine_mode == "cg1":
                feed = torch.sigmoid(z) * se + routed
            else:
                c = torch.softmax(z, dim=1)
                feed = c[:, :1] * se + c[:, 1:2] * routed
    out = h_mh_cur + feed
    if target is None:
        loss = out.mean()
    else:
        loss = ((out - target) ** 2).sum() / t
    return loss + aux_coeff * aux, out


def pair_grads(params_np: Dict[str, np.ndarray], tokens_np, **kw):
    """Gradients of pair_loss w.r.t. every parameter (float64 numpy)."""
    p = {n: torch.tensor(np.asarray(v, dtype=np.float64), requires_grad=True)
         for n, v in params_np.items()}
    loss, _ = pair_loss(p, torch.tensor(np.asarray(tokens_np, dtype=np.float64)), **kw)
    loss.backward()
    return float(loss.detach()), {n: (t.grad.numpy() if t.grad is not None else np.zeros_like(params_np[n]))
                         for n, t in p.items()}
