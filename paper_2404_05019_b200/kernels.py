"""Torch-tensor wrappers over the C ABI (one function per libscmoe entry).

All tensors must be contiguous CUDA tensors on an sm_100 device; every call is
asynchronous on the current stream (or `stream`).  Shapes follow
include/scmoe.h.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib
from ._lib import check, dtype_code, ensure_device, lib, ptr, stream_ptr


def _c(t: torch.Tensor, name: str) -> torch.Tensor:
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def expert_quota(capacity_factor: float, n_tokens: int, k: int, n_experts: int) -> int:
    """int(ceil(cf * T * k / N)) in float64, as gating.expert_quota
    (gating.py:134-135)."""
    return int(math.ceil(capacity_factor * n_tokens * k / n_experts))


@dataclass
class GateOut:
    logits: torch.Tensor    # (T, N) fp32
    indices: torch.Tensor   # (T, k) int32
    weights: torch.Tensor   # (T, k) fp32
    slots: torch.Tensor     # (T, k) int32
    dropped: torch.Tensor   # (T, k) uint8
    counts: torch.Tensor    # (N,) int32, pre-drop
    prob_sum: torch.Tensor  # (N,) fp32, sum_t softmax(logits)[t]
    quota: int


def gate_split_weights(w_gate_t: torch.Tensor, stream=None) -> Optional[torch.Tensor]:
    """3-part bf16 split of the fp32 gate weights for the tensor-core gate, or
    None when that path does not apply (N > 16 or d < 64)."""
    N, d = w_gate_t.shape
    nbytes = lib().scmoe_gate_split_bytes(N, d)
    if nbytes == 0:
        return None
    blob = torch.empty(nbytes, device=w_gate_t.device, dtype=torch.uint8)
    check(lib().scmoe_gate_split_weights(ptr(_c(w_gate_t, "w_gate_t")), N, d, ptr(blob),
                                         stream_ptr(stream)))
    return blob


def gate_topk(x: torch.Tensor, w_gate_t: torch.Tensor, k: int, quota: int,
              w_noise_t: Optional[torch.Tensor] = None, eps: Optional[torch.Tensor] = None,
              exclude: Optional[torch.Tensor] = None, w_split: Optional[torch.Tensor] = None,
              sync: Optional[torch.Tensor] = None, stream=None) -> GateOut:
    """K1/K1b: logits, top-k, masked-softmax weights and capacity slots.
    `w_split` (from gate_split_weights) skips the per-call weight split;
    `sync` (>= 2 int32, zeroed once, left zero by every call; one stream per
    sync) replaces the per-call counter memset."""
    ensure_device(x)
    if x.dim() != 2 or x.stride(1) != 1:
        raise ValueError("x must be a row-major (T, d) matrix")
    T, d = x.shape
    N = w_gate_t.shape[0]
    if w_gate_t.shape != (N, d) or w_gate_t.dtype != torch.float32:
        raise ValueError(f"w_gate_t must be fp32 ({N}, {d})")
    dev = x.device
    logits = torch.empty(T, N, device=dev, dtype=torch.float32)
    indices = torch.empty(T, k, device=dev, dtype=torch.int32)
    weights = torch.empty(T, k, device=dev, dtype=torch.float32)
    slots = torch.empty(T, k, device=dev, dtype=torch.int32)
    dropped = torch.empty(T, k, device=dev, dtype=torch.uint8)
    counts = torch.empty(N, device=dev, dtype=torch.int32)
    prob_sum = torch.empty(N, device=dev, dtype=torch.float32)
    ws_bytes = lib().scmoe_gate_workspace_bytes(T, N, d)
    ws = torch.empty(ws_bytes, device=dev, dtype=torch.uint8)
    if eps is not None:
        eps = _c(eps.to(torch.float32), "eps")
    if exclude is not None:
        exclude = _c(exclude.to(torch.int32).reshape(-1), "exclude")
    if sync is not None and (sync.dtype != torch.int32 or sync.numel() < 2 or
                             sync.device != x.device):
        raise ValueError("sync must be >= 2 int32 words on the tokens' device")
    if w_noise_t is not None:
        w_split = None
    check(lib().scmoe_gate_topk_ex(
        ptr(x), dtype_code(x.dtype), x.stride(0), ptr(_c(w_gate_t, "w_gate_t")), ptr(w_split),
        ptr(w_noise_t), ptr(eps), ptr(exclude), T, d, N, k, quota,
        ptr(logits), ptr(indices), ptr(weights), ptr(slots), ptr(dropped), ptr(counts),
        ptr(prob_sum), ptr(ws), ws_bytes, ptr(sync), stream_ptr(stream)))
    return GateOut(logits, indices, weights, slots, dropped, counts, prob_sum, quota)


def dispatch(x: torch.Tensor, indices: torch.Tensor, slots: torch.Tensor, n_experts: int,
             capacity: int, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """K2: capacity-slotted buffer (n_experts, capacity, d)."""
    ensure_device(x)
    T, d = x.shape
    k = indices.shape[1]
    if out is None:
        out = torch.empty(n_experts, capacity, d, device=x.device, dtype=x.dtype)
    check(lib().scmoe_dispatch(ptr(x), dtype_code(x.dtype), x.stride(0), T, d, k,
                               ptr(_c(indices, "indices")), ptr(_c(slots, "slots")), capacity,
                               ptr(out), stream_ptr(stream)))
    return out


def grouped_gemm(a: torch.Tensor, wt: torch.Tensor, bias: Optional[torch.Tensor],
                 group_rows: Optional[torch.Tensor] = None, rows_clip: int = 0,
                 gelu: bool = False, out: Optional[torch.Tensor] = None,
                 residual: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """out[g] = epi(a[g] @ wt[g % W]^T + bias[g % W]) (+ residual[g]) on rows < rows(g).

    a: (G, C, K) or (C, K); wt: (W, N, K) or (N, K); bias fp32 (W, N)/(N,).
    """
    ensure_device(a)
    a3 = a if a.dim() == 3 else a.unsqueeze(0)
    w3 = wt if wt.dim() == 3 else wt.unsqueeze(0)
    G, C, K = a3.shape
    W, N, K2 = w3.shape
    if K2 != K:
        raise ValueError(f"inner dims differ: {K} vs {K2}")
    if a.dtype != wt.dtype:
        raise ValueError("a and wt must share a dtype")
    if out is None:
        out = torch.empty(G, C, N, device=a.device, dtype=a.dtype)
    if bias is not None and bias.dtype != torch.float32:
        raise ValueError("bias must be fp32")
    if residual is not None:
        _c(residual, "residual")
        if residual.numel() != out.numel() or residual.dtype != out.dtype:
            raise ValueError("residual must match the output's shape and dtype")
    check(lib().scmoe_grouped_gemm(
        ptr(_c(a3, "a")), dtype_code(a.dtype), ptr(_c(w3, "wt")), ptr(bias), ptr(residual),
        ptr(out), G, W, C,
        ptr(group_rows), rows_clip, N, K, _lib.EPI_BIAS_GELU if gelu else _lib.EPI_BIAS,
        stream_ptr(stream)))
    return out if a.dim() == 3 else out.squeeze(0)


def expert_ffn(x: torch.Tensor, w1t: torch.Tensor, b1: torch.Tensor, w2t: torch.Tensor,
               b2: torch.Tensor, group_rows: Optional[torch.Tensor] = None, rows_clip: int = 0,
               hidden: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
               residual: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """expert_forward (arch.py:349-351) for every group: gelu(x W1 + b1) W2 + b2."""
    ensure_device(x)
    x3 = x if x.dim() == 3 else x.unsqueeze(0)
    w13 = w1t if w1t.dim() == 3 else w1t.unsqueeze(0)
    w23 = w2t if w2t.dim() == 3 else w2t.unsqueeze(0)
    G, C, d = x3.shape
    W, h, _ = w13.shape
    if hidden is None:
        hidden = torch.empty(G, C, h, device=x.device, dtype=x.dtype)
    if out is None:
        out = torch.empty(G, C, d, device=x.device, dtype=x.dtype)
    if residual is not None:
        _c(residual, "residual")
        if residual.numel() != out.numel() or residual.dtype != out.dtype:
            raise ValueError("residual must match the output's shape and dtype")
    check(lib().scmoe_expert_ffn(
        ptr(_c(x3, "x")), dtype_code(x.dtype), ptr(_c(w13, "w1t")), ptr(b1), ptr(_c(w23, "w2t")),
        ptr(b2), ptr(residual), ptr(hidden), ptr(out), G, W, C, ptr(group_rows), rows_clip, d, h,
        stream_ptr(stream)))
    return out if x.dim() == 3 else out.view(C, d)


def combine(expert_out: torch.Tensor, indices: torch.Tensor, slots: torch.Tensor,
            weights: torch.Tensor, capacity: int, se_out: Optional[torch.Tensor] = None,
            mode: str = "direct_add", x_cur: Optional[torch.Tensor] = None,
            w_cg: Optional[torch.Tensor] = None, residual: Optional[torch.Tensor] = None,
            out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """K5: routed gather-sum + combination gate + optional residual."""
    ensure_device(expert_out)
    for name, t in (("se_out", se_out), ("x_cur", x_cur), ("residual", residual), ("w_cg", w_cg)):
        if t is not None:
            _c(t, name)
    T, k = indices.shape
    d = expert_out.shape[-1]
    if out is None:
        out = torch.empty(T, d, device=expert_out.device, dtype=expert_out.dtype)
    check(lib().scmoe_combine(
        ptr(se_out), ptr(_c(expert_out, "expert_out")), ptr(x_cur), ptr(w_cg),
        _lib.COMBINE_MODES[mode], ptr(residual), ptr(indices), ptr(slots), ptr(weights),
        capacity, T, d, k, dtype_code(expert_out.dtype), ptr(out), stream_ptr(stream)))
    return out


def set_gemm_mode(mode: int) -> None:
    """0 = auto, 1 = force the 1-SM tcgen05 kernel, 2 = force the 2-SM kernel."""
    check(lib().scmoe_set_gemm_mode(mode))


_SM_BUDGET = [0]


class gemm_sm_budget:
    """Context manager: persistent GEMMs launched inside use at most `sms`
    SMs (None / 0 = all) — room for a concurrent exchange kernel or a
    concurrent GEMM.  Nested budgets take the smaller; the previous budget is
    restored on exit."""

    def __init__(self, sms: Optional[int]):
        self.sms = int(sms or 0)

    def __enter__(self):
        self.prev = _SM_BUDGET[0]
        new = min(self.sms, self.prev) if (self.sms and self.prev) else (self.sms or self.prev)
        _SM_BUDGET[0] = new
        check(lib().scmoe_set_gemm_sm_budget(new))
        return self

    def __exit__(self, *exc):
        _SM_BUDGET[0] = self.prev
        check(lib().scmoe_set_gemm_sm_budget(self.prev))
        return False


def set_gemm_epilogue_warps(e: int) -> None:
    """0 = auto (16 for small-K elementwise-heavy tiles), 8 or 16 forced."""
    check(lib().scmoe_set_gemm_epilogue_warps(e))


def set_gemm_flags(flags: int) -> None:
    """Experiment flags of the GEMM (A/B scripts): bit 0 row-per-thread
    epilogue operand loads, bit 3 no programmatic dependent launch, bit 4
    row-per-thread fp32 split-K partial stores."""
    check(lib().scmoe_set_gemm_flags(flags))


def set_gemm_tile_n(bn: int) -> None:
    """0 = auto, 128 or 256 = force the tcgen05 tile width (N per tile)."""
    check(lib().scmoe_set_gemm_tile_n(bn))


# ---------------------------------------------------------------------------
# training-side entries (K7)


def grouped_gemm_ex(a: torch.Tensor, w: torch.Tensor, w_layout: int, out_cols: int,
                    bias: Optional[torch.Tensor] = None, residual: Optional[torch.Tensor] = None,
                    aux_in: Optional[torch.Tensor] = None, aux_out: Optional[torch.Tensor] = None,
                    epilogue: int = _lib.EPI_BIAS, group_rows: Optional[torch.Tensor] = None,
                    rows_clip: int = 0, zero_tail: bool = False,
                    out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """out[g] = epi(a[g] @ Wg + bias) with Wg = w[g % W]^T (W_NK) or w[g % W] (W_KN)."""
    ensure_device(a)
    a3 = a if a.dim() == 3 else a.unsqueeze(0)
    w3 = w if w.dim() == 3 else w.unsqueeze(0)
    G, C, K = a3.shape
    W = w3.shape[0]
    k_in = w3.shape[2] if w_layout == _lib.W_NK else w3.shape[1]
    n_out = w3.shape[1] if w_layout == _lib.W_NK else w3.shape[2]
    if k_in != K or n_out != out_cols:
        raise ValueError(f"weight shape {tuple(w3.shape)} does not match a {tuple(a3.shape)} -> {out_cols}")
    if out is None:
        out = torch.empty(G, C, n_out, device=a.device, dtype=a.dtype)
    elif out.dtype != a.dtype or out.numel() != G * C * n_out:
        raise ValueError("out must have the operand dtype and (groups, rows, out_cols) elements")
    for name, t in (("residual", residual), ("aux_in", aux_in), ("aux_out", aux_out)):
        if t is not None:
            _c(t, name)
            if t.numel() != out.numel():
                raise ValueError(f"{name} must match the output's shape")
            if t.dtype != a.dtype:     # the C side reads it with a's element type
                raise ValueError(f"{name} dtype {t.dtype} != operand dtype {a.dtype}")
    check(lib().scmoe_grouped_gemm_ex(
        ptr(_c(a3, "a")), dtype_code(a.dtype), ptr(_c(w3, "w")), w_layout, ptr(bias),
        ptr(residual), ptr(aux_in), ptr(aux_out), ptr(out), G, W, C, ptr(group_rows), rows_clip,
        n_out, K, epilogue, 1 if zero_tail else 0, stream_ptr(stream)))
    return out if a.dim() == 3 else out.view(C, n_out)


def grouped_wgrad(a: torch.Tensor, b: torch.Tensor, n_wgroups: int = 1,
                  group_rows: Optional[torch.Tensor] = None, rows_clip: int = 0, splits: int = 0,
                  out: Optional[torch.Tensor] = None, stream=None,
                  out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """out[w] = sum_{g = w mod W} a[g, :rows(g)]^T @ b[g, :rows(g)], fp32
    accumulation; out_dtype bf16 rounds once in the split reduction (the
    parameter-dtype gradient, no conversion pass)."""
    ensure_device(a)
    a3 = a if a.dim() == 3 else a.unsqueeze(0)
    b3 = b if b.dim() == 3 else b.unsqueeze(0)
    G, C, M = a3.shape
    N = b3.shape[2]
    if b3.shape[:2] != (G, C):
        raise ValueError("a and b must share (groups, rows)")
    if out_dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("wgrad output is fp32 or bf16")
    if out is None:
        out = torch.empty(n_wgroups, M, N, device=a.device, dtype=out_dtype)
    elif out.dtype != out_dtype:
        raise ValueError("out dtype differs from out_dtype")
    ws_bytes = lib().scmoe_grouped_wgrad_workspace_bytes(n_wgroups, M, N, splits)
    if out_dtype == torch.bfloat16:
        ws_bytes = max(ws_bytes, n_wgroups * M * N * 4)
    ws = torch.empty(max(ws_bytes, 16), device=a.device, dtype=torch.uint8)
    check(lib().scmoe_grouped_wgrad_ex(
        ptr(_c(a3, "a")), ptr(_c(b3, "b")), dtype_code(a.dtype), ptr(out), dtype_code(out_dtype),
        ptr(ws), ws_bytes, G, n_wgroups, C, ptr(group_rows), rows_clip, M, N, splits,
        stream_ptr(stream)))
    return out if (a.dim() == 3 or n_wgroups > 1) else out.view(M, N)


def gather_rows(src: torch.Tensor, ids: torch.Tensor, n_rows: torch.Tensor, max_rows: int,
                out: torch.Tensor, stream=None) -> torch.Tensor:
    """out[j] = src[ids[j]] for j < min(n_rows, max_rows); src may be pinned
    host memory (the kernel reads it over the host link)."""
    ensure_device(out)
    if src.is_cuda is False and not src.is_pinned():
        raise ValueError("host-side source rows must be in pinned memory")
    row_bytes = src[0].numel() * src.element_size()
    check(lib().scmoe_gather_rows(ptr(_c(src, "src")), row_bytes, ptr(_c(ids, "ids")),
                                  ptr(n_rows), max_rows, ptr(_c(out, "out")), stream_ptr(stream)))
    return out


def sgd_update(params, grads, lr: float, stream=None) -> None:
    """p -= lr * g for every (p, g) pair in one launch (bf16 / fp32 pairs of the
    same dtype, 16-byte aligned whole vectors)."""
    n = len(params)
    if n == 0:
        return
    P = (ctypes.c_void_p * n)(*[p.data_ptr() for p in params])
    G = (ctypes.c_void_p * n)(*[g.data_ptr() for g in grads])
    N = (ctypes.c_longlong * n)(*[p.numel() for p in params])
    D = (ctypes.c_int * n)(*[dtype_code(p.dtype) for p in params])
    check(lib().scmoe_sgd_update(P, G, N, D, n, float(lr), stream_ptr(stream)))


def copy_rows(src: torch.Tensor, ids_host: torch.Tensor, n_rows: int, out: torch.Tensor,
              stream=None) -> torch.Tensor:
    """out[j] = src[ids_host[j]] for j < n_rows on the copy engine
    (cudaMemcpyAsync on `stream`); ids_host is a host int32 tensor."""
    ensure_device(out)
    if src.is_cuda is False and not src.is_pinned():
        raise ValueError("host-side source rows must be in pinned memory")
    if ids_host.is_cuda or ids_host.dtype != torch.int32:
        raise ValueError("copy_rows takes the row ids as a host int32 tensor")
    if n_rows > out.shape[0] or n_rows > ids_host.numel():
        raise ValueError("copy_rows: more rows than the output / id list holds")
    row_bytes = src[0].numel() * src.element_size()
    check(lib().scmoe_copy_rows(ptr(_c(src, "src")), row_bytes, ptr(ids_host), int(n_rows),
                                ptr(_c(out, "out")), stream_ptr(stream)))
    return out


def gate_backward(src: torch.Tensor, logits: torch.Tensor, indices: torch.Tensor,
                  weights: torch.Tensor, counts: torch.Tensor, w_gate_t: torch.Tensor,
                  d_weights: Optional[torch.Tensor] = None, d_aux: Optional[torch.Tensor] = None,
                  w_noise_t: Optional[torch.Tensor] = None, eps: Optional[torch.Tensor] = None,
                  noise_pre: Optional[torch.Tensor] = None, need_src: bool = True,
                  stream=None):
    """K7 gate backward (one pass over the tokens): returns (d_src or None,
    d_w_gate (N, d) fp32, d_w_noise (N, d) fp32 or None)."""
    ensure_device(src)
    T, d = src.shape
    N = logits.shape[1]
    k = indices.shape[1]
    noise = w_noise_t is not None
    f32 = dict(device=src.device, dtype=torch.float32)
    d_src = torch.empty_like(src) if need_src else None
    d_wg = torch.empty(N, d, **f32)
    d_wn = torch.empty(N, d, **f32) if noise else None
    ws_bytes = lib().scmoe_gate_backward_workspace_bytes(T, d, N, 1 if noise else 0)
    ws = torch.empty(max(ws_bytes, 16), device=src.device, dtype=torch.uint8)
    if d_weights is not None:
        d_weights = _c(d_weights.float(), "d_weights")
    if d_aux is not None:
        d_aux = d_aux.detach().float().reshape(1).contiguous()
    check(lib().scmoe_gate_backward(
        ptr(_c(src, "src")), dtype_code(src.dtype), T, d, N, k, ptr(_c(logits, "logits")),
        ptr(_c(indices, "indices")), ptr(_c(weights, "weights")), ptr(d_weights),
        ptr(_c(counts, "counts")), ptr(d_aux), ptr(_c(w_gate_t, "w_gate_t")), ptr(w_noise_t),
        ptr(eps), ptr(noise_pre), ptr(d_src), ptr(d_wg), ptr(d_wn), ptr(ws), ws_bytes,
        stream_ptr(stream)))
    return d_src, d_wg, d_wn


def gelu_fwd(z: torch.Tensor, group_rows: Optional[torch.Tensor] = None, rows_clip: int = 0,
             out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """h = gelu(z) (exact erf) on each group's valid rows, zero-padded tails."""
    ensure_device(z)
    z3 = z if z.dim() == 3 else z.unsqueeze(0)
    G, C, H = z3.shape
    if z.dtype != torch.bfloat16:
        raise ValueError("gelu_fwd is bf16")
    if out is None:
        out = torch.empty_like(z3)
    check(lib().scmoe_gelu_fwd(ptr(_c(z3, "z")), ptr(_c(out, "out")), G, C, H, ptr(group_rows),
                               rows_clip, stream_ptr(stream)))
    return out if z.dim() == 3 else out.view(C, H)


def gelu_fwd_grad(z: torch.Tensor, group_rows: Optional[torch.Tensor] = None,
                  rows_clip: int = 0, stream=None):
    """(gelu(z), gelu'(z)) on each group's valid rows, zero-padded tails."""
    ensure_device(z)
    z3 = z if z.dim() == 3 else z.unsqueeze(0)
    G, C, H = z3.shape
    if z.dtype != torch.bfloat16:
        raise ValueError("gelu_fwd_grad is bf16")
    h, dg = torch.empty_like(z3), torch.empty_like(z3)
    check(lib().scmoe_gelu_fwd_grad(ptr(_c(z3, "z")), ptr(h), ptr(dg), G, C, H, ptr(group_rows),
                                    rows_clip, stream_ptr(stream)))
    if z.dim() == 3:
        return h, dg
    return h.view(C, H), dg.view(C, H)


def gelu_bwd(dh: torch.Tensor, z: torch.Tensor, group_rows: Optional[torch.Tensor] = None,
             rows_clip: int = 0, bias_grad: bool = True, stream=None):
    """(dz = dh * gelu'(z) with zero-padded tails, per-group bias gradient
    sum_rows dz (G, H) fp32 or None)."""
    ensure_device(dh)
    d3 = dh if dh.dim() == 3 else dh.unsqueeze(0)
    z3 = z if z.dim() == 3 else z.unsqueeze(0)
    G, C, H = d3.shape
    if z3.shape != d3.shape or dh.dtype != torch.bfloat16 or z.dtype != torch.bfloat16:
        raise ValueError("gelu_bwd: dh and z must be bf16 of one shape")
    dz = torch.empty_like(d3)
    db = torch.empty(G, H, device=dh.device, dtype=torch.float32) if bias_grad else None
    ws_bytes = lib().scmoe_gelu_bwd_workspace_bytes(G, C, H) if bias_grad else 0
    ws = torch.empty(max(ws_bytes, 16), device=dh.device, dtype=torch.uint8)
    check(lib().scmoe_gelu_bwd(ptr(_c(d3, "dh")), ptr(_c(z3, "z")), ptr(dz), ptr(db), G, C, H,
                               ptr(group_rows), rows_clip, ptr(ws), ws_bytes, stream_ptr(stream)))
    return (dz if dh.dim() == 3 else dz.view(C, H)), db


def window_attention_supported(seq_len: int, head_dim: int) -> bool:
    return bool(lib().scmoe_window_attention_supported(seq_len, head_dim))


def window_attention_fwd(qkv: torch.Tensor, n_heads: int, seq_len: int, scale: float,
                         causal: bool = False, need_lse: bool = True, stream=None):
    """Windowed attention on the packed (T, 3d) projection -> (out (T, d),
    lse (T, H) fp32 base-2 or None)."""
    ensure_device(qkv)
    T, d3 = qkv.shape
    d = d3 // 3
    out = torch.empty(T, d, device=qkv.device, dtype=qkv.dtype)
    lse = torch.empty(T, n_heads, device=qkv.device, dtype=torch.float32) if need_lse else None
    if qkv.dtype != torch.bfloat16:
        raise ValueError("window attention is bf16")
    check(lib().scmoe_window_attention_fwd(ptr(_c(qkv, "qkv")), T, n_heads, d // n_heads, seq_len,
                                           float(scale), 1 if causal else 0, ptr(out), ptr(lse),
                                           stream_ptr(stream)))
    return out, lse


def window_attention_bwd(qkv: torch.Tensor, out: torch.Tensor, dout: torch.Tensor,
                         lse: torch.Tensor, n_heads: int, seq_len: int, scale: float,
                         causal: bool = False, stream=None) -> torch.Tensor:
    """dqkv (T, 3d) in the packed layout."""
    ensure_device(qkv)
    T, d3 = qkv.shape
    dqkv = torch.empty_like(qkv)
    check(lib().scmoe_window_attention_bwd(
        ptr(_c(qkv, "qkv")), ptr(_c(out, "out")), ptr(_c(dout, "dout")), ptr(_c(lse, "lse")), T,
        n_heads, d3 // 3 // n_heads, seq_len, float(scale), 1 if causal else 0, ptr(dqkv),
        stream_ptr(stream)))
    return dqkv


_ONES = {}


def bias_grad(dy: torch.Tensor, n_wgroups: int = 1, group_rows: Optional[torch.Tensor] = None,
              rows_clip: int = 0, stream=None) -> torch.Tensor:
    """Bias gradient sum_{g = w mod W} sum_{r < rows(g)} dy[g, r, :] as the
    tensor-core weight gradient 1^T dy (K7 wgrad with an all-ones (C, 8)
    operand): dy is read once, split-K across the GPU, the zero-padded tails
    of dy keep the partial last 64-row block exact.  Returns (W, N) fp32."""
    ensure_device(dy)
    d3 = dy if dy.dim() == 3 else dy.unsqueeze(0)
    G, C, N = d3.shape
    key = (d3.device, d3.dtype, G, C)
    ones = _ONES.get(key)
    if ones is None:
        ones = torch.ones(G, C, 8, device=d3.device, dtype=d3.dtype)
        _ONES[key] = ones
    out = grouped_wgrad(ones, d3, n_wgroups=n_wgroups, group_rows=group_rows,
                        rows_clip=rows_clip, stream=stream)
    return out.view(n_wgroups, 8, N)[:, 0, :]


def zero_tails(buf: torch.Tensor, group_rows: torch.Tensor, rows_clip: int = 0, align: int = 64,
               stream=None) -> torch.Tensor:
    ensure_device(buf)
    b3 = buf if buf.dim() == 3 else buf.unsqueeze(0)
    G, C, D = b3.shape
    check(lib().scmoe_zero_tails(ptr(_c(b3, "buf")), dtype_code(buf.dtype), G, C, D,
                                 ptr(group_rows), rows_clip, align, stream_ptr(stream)))
    return buf


def grouped_colsum(x: torch.Tensor, group_rows: Optional[torch.Tensor] = None, rows_clip: int = 0,
                   stream=None) -> torch.Tensor:
    ensure_device(x)
    x3 = x if x.dim() == 3 else x.unsqueeze(0)
    G, C, D = x3.shape
    out = torch.empty(G, D, device=x.device, dtype=torch.float32)
    ws_bytes = lib().scmoe_grouped_colsum_workspace_bytes(G, C, D)
    ws = torch.empty(ws_bytes, device=x.device, dtype=torch.uint8)
    check(lib().scmoe_grouped_colsum(ptr(_c(x3, "x")), dtype_code(x.dtype), G, C, D,
                                     ptr(group_rows), rows_clip, ptr(out), ptr(ws), ws_bytes,
                                     stream_ptr(stream)))
    return out if x.dim() == 3 else out.view(D)


def gate_aux_loss(counts: torch.Tensor, prob_sum: torch.Tensor, n_tokens: int, k: int,
                  stream=None) -> torch.Tensor:
    """Balance loss N * sum_e f_e P_e from the gate kernel's counts and
    probability sums, one launch (arch.py:436-439)."""
    ensure_device(counts)
    if counts.dtype != torch.int32 or prob_sum.dtype != torch.float32 or \
            prob_sum.numel() != counts.numel():
        raise ValueError("aux loss needs int32 counts and fp32 prob_sum of one length")
    aux = torch.empty((), device=counts.device, dtype=torch.float32)
    check(lib().scmoe_gate_aux_loss(ptr(_c(counts, "counts")), ptr(_c(prob_sum, "prob_sum")),
                                    n_tokens, counts.shape[0], k, ptr(aux), stream_ptr(stream)))
    return aux


def mean_f32(x: torch.Tensor, stream=None) -> torch.Tensor:
    """mean of every element of x (bf16 / fp32) accumulated in fp32, as a
    0-dim fp32 tensor; deterministic, two launches, no memset."""
    ensure_device(x)
    out = torch.empty((), device=x.device, dtype=torch.float32)
    ws_bytes = lib().scmoe_mean_workspace_bytes()
    ws = torch.empty(ws_bytes, device=x.device, dtype=torch.uint8)
    check(lib().scmoe_mean(ptr(_c(x, "x")), dtype_code(x.dtype), x.numel(), ptr(out), ptr(ws),
                           ws_bytes, stream_ptr(stream)))
    return out


def fill_div(out: torch.Tensor, src: torch.Tensor, div: float, stream=None) -> torch.Tensor:
    """out[:] = (src / div) in out's dtype, src a one-element fp32 device tensor."""
    ensure_device(out)
    if src.dtype != torch.float32 or src.numel() != 1:
        raise ValueError("src must be a one-element fp32 tensor")
    check(lib().scmoe_fill_div(ptr(_c(out, "out")), dtype_code(out.dtype), out.numel(),
                               ptr(_c(src, "src")), float(div), stream_ptr(stream)))
    return out


def grouped_colsum2(x0: torch.Tensor, x1: torch.Tensor, group_rows: Optional[torch.Tensor] = None,
                    rows_clip: int = 0, stream=None):
    """(grouped_colsum(x0), grouped_colsum(x1)) for two matrices with the same
    groups and dtype, one launch per pass."""
    ensure_device(x0)
    a = x0 if x0.dim() == 3 else x0.unsqueeze(0)
    b = x1 if x1.dim() == 3 else x1.unsqueeze(0)
    G, C, D0 = a.shape
    if b.shape[:2] != (G, C) or b.dtype != a.dtype:
        raise ValueError("grouped_colsum2 needs the same groups, rows and dtype")
    D1 = b.shape[2]
    out = torch.empty(G * (D0 + D1), device=x0.device, dtype=torch.float32)
    o0, o1 = out[:G * D0].view(G, D0), out[G * D0:].view(G, D1)
    ws_bytes = lib().scmoe_grouped_colsum2_workspace_bytes(G, C, D0, D1)
    ws = torch.empty(ws_bytes, device=x0.device, dtype=torch.uint8)
    check(lib().scmoe_grouped_colsum2(ptr(_c(a, "x0")), ptr(_c(b, "x1")), dtype_code(a.dtype), G, C,
                                      D0, D1, ptr(group_rows), rows_clip, ptr(o0), ptr(o1),
                                      ptr(ws), ws_bytes, stream_ptr(stream)))
    return (o0 if x0.dim() == 3 else o0.view(D0)), (o1 if x1.dim() == 3 else o1.view(D1))


def dispatch_scaled(x: torch.Tensor, indices: torch.Tensor, slots: torch.Tensor, n_experts: int,
                    capacity: int, row_scale: Optional[torch.Tensor],
                    out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """dispatch with each copied row scaled by row_scale[t, j] (combine backward)."""
    ensure_device(x)
    T, d = x.shape
    k = indices.shape[1]
    if out is None:
        out = torch.empty(n_experts, capacity, d, device=x.device, dtype=x.dtype)
    if row_scale is not None:
        row_scale = _c(row_scale.to(torch.float32), "row_scale")
    check(lib().scmoe_dispatch_scaled(ptr(x), dtype_code(x.dtype), x.stride(0), T, d, k,
                                      ptr(_c(indices, "indices")), ptr(_c(slots, "slots")),
                                      capacity, ptr(row_scale), ptr(out), stream_ptr(stream)))
    return out


def pack_heads(srcs, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """(B, H, S, hd) bf16 tensors (any strides, hd contiguous) -> one
    (B, S, n, H, hd) contiguous tensor (scmoe_pack_heads)."""
    import ctypes
    b, h, s, hd = srcs[0].shape
    for t in srcs:
        ensure_device(t)
        if t.shape != srcs[0].shape or t.stride(3) != 1 or t.dtype != torch.bfloat16:
            raise ValueError("pack_heads: bf16 (B, H, S, hd) sources with contiguous hd")
    n = len(srcs)
    if out is None:
        out = torch.empty(b, s, n, h, hd, device=srcs[0].device, dtype=srcs[0].dtype)
    ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() for t in srcs])
    strides = (ctypes.c_longlong * (3 * n))(*[v for t in srcs for v in t.stride()[:3]])
    check(lib().scmoe_pack_heads(ctypes.cast(ptrs, ctypes.c_void_p),
                                 ctypes.cast(strides, ctypes.c_void_p), n, b, h, s, hd,
                                 _lib.SCMOE_BF16, ptr(out), stream_ptr(stream)))
    return out


def ffn2_combine(hidden: torch.Tensor, w2t: torch.Tensor, b2: torch.Tensor,
                 expert_out: torch.Tensor, indices: torch.Tensor, slots: torch.Tensor,
                 weights: torch.Tensor, capacity: int, residual: Optional[torch.Tensor] = None,
                 out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """The second half of shared_ffn_combine over a precomputed hidden =
    gelu(x W1 + b1): GEMM2 with the direct-add combine in its epilogue."""
    ensure_device(hidden)
    T, h = hidden.shape
    d = w2t.shape[-2]
    if out is None:
        out = torch.empty(T, d, device=hidden.device, dtype=hidden.dtype)
    if residual is not None:
        _c(residual, "residual")
    check(lib().scmoe_ffn2_combine(
        ptr(_c(hidden, "hidden")), dtype_code(hidden.dtype), ptr(_c(w2t, "w2t")), ptr(b2),
        ptr(residual), ptr(_c(expert_out, "expert_out")), ptr(_c(indices, "indices")),
        ptr(_c(slots, "slots")), ptr(_c(weights, "weights")), capacity, indices.shape[1],
        ptr(out), T, d, h, stream_ptr(stream)))
    return out


def shared_ffn_combine(x: torch.Tensor, w1t: torch.Tensor, b1: torch.Tensor, w2t: torch.Tensor,
                       b2: torch.Tensor, expert_out: torch.Tensor, indices: torch.Tensor,
                       slots: torch.Tensor, weights: torch.Tensor, capacity: int,
                       residual: Optional[torch.Tensor] = None,
                       out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Shared expert on x with the direct-add ScMoE combine fused into its
    GEMM2 epilogue (scmoe_shared_ffn_combine): = combine(SE(x), routed) + res."""
    ensure_device(x)
    T, d = x.shape
    h = w1t.shape[-2]
    hidden = torch.empty(T, h, device=x.device, dtype=x.dtype)
    if out is None:
        out = torch.empty(T, d, device=x.device, dtype=x.dtype)
    if residual is not None:
        _c(residual, "residual")
    check(lib().scmoe_shared_ffn_combine(
        ptr(_c(x, "x")), dtype_code(x.dtype), ptr(_c(w1t, "w1t")), ptr(b1), ptr(_c(w2t, "w2t")),
        ptr(b2), ptr(residual), ptr(_c(expert_out, "expert_out")), ptr(_c(indices, "indices")),
        ptr(_c(slots, "slots")), ptr(_c(weights, "weights")), capacity, indices.shape[1],
        ptr(hidden), ptr(out), T, d, h, stream_ptr(stream)))
    return out
