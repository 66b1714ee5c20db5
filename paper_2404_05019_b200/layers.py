"""Torch modules of the ScMoE layer (arXiv 2404.05019) on the sm_100a kernels.

API mirror of the reference (`/root/reference/pkg/src/scmoelab/`):

  reference                               here
  --------------------------------------  -----------------------------------------
  gating.CapacityConfig  (gating.py:39)   CapacityConfig
  gating.GateDecision    (gating.py:51)   GateDecision (+ slots, counts, prob_sum)
  gating.GateParams + gate_logits /       Top1Gate(d_model, n_experts, k=1,
   select_topk / apply_capacity             noise_enabled=False) — one kernel (K1)
   (gating.py:20-156)
  arch.expert_forward    (arch.py:349)    SharedExpert(d_model, d_hidden) (K4)
  arch.combine           (arch.py:380)    fused into the combine kernel (K5)
  arch.moe_shared        (arch.py:496)    ScMoELayer(...).forward(x_cur, routed_src)
  arch.moe_standard k=2  (arch.py:489)    Top2MoELayer(...).forward(x)
  arch.MoEReplay         (arch.py:315)    MoEReplay (pinned indices / drops / eps)

Constructor arguments are the reference's ModelConfig / dataclass fields
(d_model, d_hidden, n_experts, k_routed, combine_mode, capacity_factor,
noise_enabled); `forward` returns (out, decision, aux) like moe_shared /
moe_standard.  Everything runs on the GPU through libscmoe (no CPU fallback).
Weights are stored K-major (w1t = W1^T, w2t = W2^T) for the tcgen05 tiles.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch
from torch import nn

from . import kernels as K
from ._lib import MAX_EXPERTS, MAX_K

COMBINE_MODES = ("direct_add", "cg1", "cg2")


class ConfigError(ValueError):
    """Mirror of arch.ConfigError (arch.py:31-32)."""


@dataclass
class CapacityConfig:
    """gating.CapacityConfig (gating.py:39-48)."""
    capacity_factor: float = 2.0
    policy: str = "drop-overflow"

    def __post_init__(self):
        if self.capacity_factor <= 0:
            raise ValueError("capacity_factor must be > 0")
        if self.policy != "drop-overflow":
            raise ValueError(f"unknown capacity policy {self.policy!r}")


@dataclass
class MoEReplay:
    """arch.MoEReplay (arch.py:315-322): pinned noise draws and routing; the
    *_prev fields are the preceding gating of dual gating (DGMoE)."""
    eps: Optional[object] = None
    indices: Optional[object] = None
    dropped: Optional[object] = None
    eps_prev: Optional[object] = None
    indices_prev: Optional[object] = None
    dropped_prev: Optional[object] = None


@dataclass
class GateDecision:
    """gating.GateDecision (gating.py:51-90) as device tensors, plus the
    capacity slot of every selection and the per-expert statistics the
    balance loss needs."""
    logits: torch.Tensor              # (T, N) fp32
    indices: torch.Tensor             # (T, k) int32, rank order = logit order
    weights: torch.Tensor             # (T, k) fp32 masked-softmax weights
    dropped: torch.Tensor             # (T, k) bool
    slots: torch.Tensor               # (T, k) int32 capacity slot
    counts: torch.Tensor              # (N,) int32 pre-drop selections
    prob_sum: torch.Tensor            # (N,) fp32 sum of full-softmax probs
    quota: int                        # ceil(cf*T*k/N)
    capacity: int                     # rows per expert in the dispatch buffer
    eps: Optional[torch.Tensor] = None

    @property
    def n_tokens(self) -> int:
        return self.logits.shape[0]

    @property
    def n_experts(self) -> int:
        return self.logits.shape[1]

    @property
    def k(self) -> int:
        return self.indices.shape[1]

    def support_mask(self) -> torch.Tensor:
        m = torch.zeros_like(self.logits, dtype=torch.bool)
        m.scatter_(1, self.indices.long(), True)
        return m

    def keep_mask(self) -> torch.Tensor:
        m = torch.zeros_like(self.logits)
        m.scatter_(1, self.indices.long(), (~self.dropped).to(m.dtype))
        return m

    def kept_counts(self) -> torch.Tensor:
        """Rows each expert holds in the dispatch buffer."""
        if self.capacity == self.quota:
            return torch.clamp(self.counts, max=self.quota)
        keep = (~self.dropped).reshape(-1).to(torch.float32)
        return torch.bincount(self.indices.reshape(-1).long(), weights=keep,
                              minlength=self.n_experts).to(torch.int32)

    def aux_loss(self) -> torch.Tensor:
        """N * sum_i f_i P_i (arch.py:436-439 / gating.py:159-170), one kernel."""
        return K.gate_aux_loss(self.counts, self.prob_sum, self.n_tokens, self.k)

    def to_numpy(self) -> dict:
        return dict(logits=self.logits.double().cpu().numpy(),
                    indices=self.indices.long().cpu().numpy(),
                    weights=self.weights.double().cpu().numpy(),
                    dropped=self.dropped.cpu().numpy().astype(bool),
                    slots=self.slots.long().cpu().numpy(),
                    eps=None if self.eps is None else self.eps.double().cpu().numpy())


def _as_tensor(a, device, dtype):
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype)
    return torch.as_tensor(np.asarray(a), device=device, dtype=dtype)


def _normal_(t: torch.Tensor, scale: float, generator: Optional[torch.Generator]):
    with torch.no_grad():
        tmp = torch.randn(t.shape, generator=generator, dtype=torch.float32, device=t.device)
        t.copy_(tmp * scale)
    return t


# ---------------------------------------------------------------------------
# gate


class Top1Gate(nn.Module):
    """Top-k softmax gate (k=1 for ScMoE) with capacity slots: GateParams +
    gate_logits + select_topk + apply_capacity (gating.py:20-156) as one
    kernel pass.  w_gate is stored transposed (N, d) in fp32."""

    def __init__(self, d_model: int, n_experts: int, k: int = 1, noise_enabled: bool = False,
                 capacity_factor: float = 2.0, device=None, generator=None):
        super().__init__()
        if not 1 <= n_experts <= MAX_EXPERTS:
            raise ConfigError(f"n_experts={n_experts} out of [1, {MAX_EXPERTS}]")
        if not 1 <= k <= min(n_experts, MAX_K):
            raise ValueError(f"k={k} out of range for N={n_experts}")
        self.d_model, self.n_experts, self.k = d_model, n_experts, k
        self.noise_enabled = noise_enabled
        self.capacity = CapacityConfig(capacity_factor)
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.w_gate_t = nn.Parameter(torch.empty(n_experts, d_model, device=dev), requires_grad=False)
        self.w_noise_t = nn.Parameter(torch.empty(n_experts, d_model, device=dev), requires_grad=False)
        self.reset_parameters(generator)

    def reset_parameters(self, generator=None):
        s = 1.0 / math.sqrt(self.d_model)     # init_params scale (arch.py:169)
        _normal_(self.w_gate_t, s, generator)
        _normal_(self.w_noise_t, s, generator)

    def quota(self, n_tokens: int) -> int:
        return K.expert_quota(self.capacity.capacity_factor, n_tokens, self.k, self.n_experts)

    def presplit(self, x_src: torch.Tensor) -> Optional[torch.Tensor]:
        """Inference only: the tensor-core gate's split weights, cached per
        weight version (in-place updates bump `_version`).  A CUDA graph
        captured with a valid cache replays with that split, so weights must
        not change between replays of such a graph (training steps — grad
        mode — always split inside the call)."""
        w = self.w_gate_t
        if (torch.is_grad_enabled() or self.noise_enabled or x_src.dtype != torch.bfloat16
                or w.requires_grad):
            return None
        key = (w.data_ptr(), w._version)
        if getattr(self, "_split_key", None) != key:
            self._split = K.gate_split_weights(w)
            self._split_key = key
        return self._split

    def _sync_words(self, device) -> torch.Tensor:
        """The tensor-core gate's cross-CTA counter, kept per gate (zeroed
        once here, left zero by every launch): no memset node per call.  A
        gate's launches never overlap in time (one stream per forward)."""
        w = getattr(self, "_sync", None)
        if w is None or w.device != device:
            w = torch.zeros(4, device=device, dtype=torch.int32)
            self._sync = w
        return w

    def forward(self, x_src: torch.Tensor, eps: Optional[torch.Tensor] = None,
                generator: Optional[torch.Generator] = None, replay: Optional[MoEReplay] = None,
                stream=None) -> GateDecision:
        t = x_src.shape[0]
        if t == 0:
            raise ValueError("empty token batch")
        if x_src.shape[1] != self.d_model:
            raise ValueError(f"x has width {x_src.shape[1]}, expected {self.d_model}")
        if replay is not None and replay.eps is not None:
            eps = _as_tensor(replay.eps, x_src.device, torch.float32)
        if self.noise_enabled and eps is None:
            eps = torch.randn(t, self.n_experts, device=x_src.device, generator=generator)
        quota = self.quota(t)
        g = K.gate_topk(x_src, self.w_gate_t, self.k, quota,
                        w_noise_t=self.w_noise_t if self.noise_enabled else None,
                        eps=eps if self.noise_enabled else None,
                        w_split=self.presplit(x_src), sync=self._sync_words(x_src.device),
                        stream=stream)
        # uint8 0/1 flags reinterpreted as bool: no conversion kernel
        dec = GateDecision(g.logits, g.indices, g.weights, g.dropped.view(torch.bool), g.slots,
                           g.counts, g.prob_sum, quota, quota,
                           eps if self.noise_enabled else None)
        if replay is not None and replay.indices is not None:
            dec = _pin_routing(dec, replay)
        return dec


def _pin_routing(dec: GateDecision, replay: MoEReplay) -> GateDecision:
    """Replay pinned indices / drop flags (arch.py:395-402, 474-477): weights
    are the masked softmax of the live logits over the pinned support; kept
    selections get consecutive slots per expert in token-major order.  This is
    a debugging / gradient-check hook, not the throughput path (it syncs once
    to size the dispatch buffer)."""
    dev = dec.logits.device
    idx = _as_tensor(replay.indices, dev, torch.int64)
    t, k = idx.shape
    if replay.dropped is None:
        drop = torch.zeros(t, k, dtype=torch.bool, device=dev)
    else:
        drop = _as_tensor(replay.dropped, dev, torch.bool)
    sel = dec.logits.gather(1, idx)
    w = torch.softmax(sel, dim=1)
    n = dec.n_experts
    flat = idx.reshape(-1)
    keep = (~drop).reshape(-1)
    onehot = torch.nn.functional.one_hot(flat, n).to(torch.int32) * keep[:, None].to(torch.int32)
    before = torch.cumsum(onehot, dim=0) - onehot
    slots = before.gather(1, flat[:, None]).reshape(t, k).to(torch.int32)
    kept = onehot.sum(dim=0)
    cap = max(int(kept.max().item()) if kept.numel() else 1, 1)
    slots = torch.where(drop, torch.full_like(slots, cap), slots)
    counts = torch.bincount(flat, minlength=n).to(torch.int32)
    return GateDecision(dec.logits, idx.to(torch.int32), w.float(), drop, slots, counts,
                        dec.prob_sum, dec.quota, cap, dec.eps)


def _with_capacity(dec: GateDecision, cap: int) -> GateDecision:
    """The same decision in a dispatch buffer of `cap` rows per expert
    (cap >= every kept count): dropped selections point past the new end."""
    if cap == dec.capacity:
        return dec
    slots = torch.where(dec.dropped, torch.full_like(dec.slots, cap), dec.slots)
    return GateDecision(dec.logits, dec.indices, dec.weights, dec.dropped, slots, dec.counts,
                        dec.prob_sum, dec.quota, cap, dec.eps)


def _agree_capacity(dec: GateDecision, group) -> GateDecision:
    """Pinned routing under expert parallelism: the dispatch capacity is the
    max over ranks of the pinned kept counts, so the equal-split exchanges
    agree on the block size."""
    import torch.distributed as dist
    caps = [None] * dist.get_world_size(group)
    dist.all_gather_object(caps, int(dec.capacity), group=group)
    return _with_capacity(dec, max(caps))


# ---------------------------------------------------------------------------
# experts


class SharedExpert(nn.Module):
    """expert_forward (arch.py:349-351) as a dense FFN: gelu(x W1 + b1) W2 + b2.
    Used for the shared expert (x_cur) and for Block-MLP."""

    def __init__(self, d_model: int, d_hidden: int, dtype=torch.bfloat16, device=None,
                 generator=None):
        super().__init__()
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.d_model, self.d_hidden = d_model, d_hidden
        self.w1t = nn.Parameter(torch.empty(d_hidden, d_model, device=dev, dtype=dtype), requires_grad=False)
        self.b1 = nn.Parameter(torch.zeros(d_hidden, device=dev), requires_grad=False)
        self.w2t = nn.Parameter(torch.empty(d_model, d_hidden, device=dev, dtype=dtype), requires_grad=False)
        self.b2 = nn.Parameter(torch.zeros(d_model, device=dev), requires_grad=False)
        self.reset_parameters(generator)

    def reset_parameters(self, generator=None):
        s = 1.0 / math.sqrt(self.d_model)     # both W1 and W2 use 1/sqrt(d) (arch.py:158-164)
        _normal_(self.w1t, s, generator)
        _normal_(self.w2t, s, generator)
        with torch.no_grad():
            self.b1.zero_()
            self.b2.zero_()

    def load_reference(self, e) -> "SharedExpert":
        """Copy an ExpertParams (w1 (d,h), b1 (1,h), w2 (h,d), b2 (1,d))."""
        dev = self.w1t.device
        with torch.no_grad():
            self.w1t.copy_(_as_tensor(np.asarray(e.w1).T, dev, self.w1t.dtype))
            self.b1.copy_(_as_tensor(np.asarray(e.b1).reshape(-1), dev, torch.float32))
            self.w2t.copy_(_as_tensor(np.asarray(e.w2).T, dev, self.w2t.dtype))
            self.b2.copy_(_as_tensor(np.asarray(e.b2).reshape(-1), dev, torch.float32))
        return self

    def forward(self, x: torch.Tensor, residual: Optional[torch.Tensor] = None,
                hidden: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                stream=None, link: Optional[dict] = None) -> torch.Tensor:
        """expert_forward(x) (+ residual, fused into the second GEMM's epilogue).
        link (training): a residual gradient of x parked by the combine is
        added in this FFN's data-gradient GEMM (training.FFNFn)."""
        if x.dtype != self.w1t.dtype:
            raise ValueError(f"input dtype {x.dtype} != expert dtype {self.w1t.dtype}")
        if torch.is_grad_enabled() and (self.w1t.requires_grad or x.requires_grad):
            from .training import FFNFn
            return FFNFn.apply(x, self.w1t, self.b1, self.w2t, self.b2, residual, None,
                               x.shape[0], link)
        return K.expert_ffn(x, self.w1t, self.b1, self.w2t, self.b2, hidden=hidden, out=out,
                            residual=residual, stream=stream)

    def forward_combine(self, x: torch.Tensor, expert_out: torch.Tensor, dec,
                        residual: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """Inference: SE(x) with the direct-add combine of the routed rows
        (+ residual) fused into the second GEMM's epilogue — bit-identical to
        forward() followed by the combine kernel."""
        return K.shared_ffn_combine(x, self.w1t, self.b1, self.w2t, self.b2, expert_out,
                                    dec.indices, dec.slots, dec.weights, dec.capacity,
                                    residual=residual, stream=stream)

    def hidden(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """Inference: gelu(x W1 + b1), the first GEMM of forward_combine (same
        kernel and epilogue: bit-identical)."""
        return K.grouped_gemm(x, self.w1t, self.b1, gelu=True, stream=stream)

    def combine_from_hidden(self, hid: torch.Tensor, expert_out: torch.Tensor, dec,
                            residual: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """forward_combine's second GEMM with the fused combine, over hidden()."""
        return K.ffn2_combine(hid, self.w2t, self.b2, expert_out, dec.indices, dec.slots,
                              dec.weights, dec.capacity, residual=residual, stream=stream)

    def can_fuse_combine(self, x: torch.Tensor, dec, combine_mode: str) -> bool:
        return (combine_mode == "direct_add" and x.dtype == torch.bfloat16 and dec.k <= 2
                and not torch.is_grad_enabled() and FUSED_COMBINE)


FUSED_COMBINE = True     # SE GEMM2 epilogue does the direct-add combine (A/B switch)


class RoutedExperts(nn.Module):
    """N stacked experts (E, h, d) / (E, d, h), evaluated only on the rows
    routed to them (the sparse equivalent of _routed_sum, arch.py:418-433)."""

    def __init__(self, n_experts: int, d_model: int, d_hidden: int, dtype=torch.bfloat16,
                 device=None, generator=None):
        super().__init__()
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.n_experts, self.d_model, self.d_hidden = n_experts, d_model, d_hidden
        self.w1t = nn.Parameter(torch.empty(n_experts, d_hidden, d_model, device=dev, dtype=dtype), requires_grad=False)
        self.b1 = nn.Parameter(torch.zeros(n_experts, d_hidden, device=dev), requires_grad=False)
        self.w2t = nn.Parameter(torch.empty(n_experts, d_model, d_hidden, device=dev, dtype=dtype), requires_grad=False)
        self.b2 = nn.Parameter(torch.zeros(n_experts, d_model, device=dev), requires_grad=False)
        self.reset_parameters(generator)

    def reset_parameters(self, generator=None):
        s = 1.0 / math.sqrt(self.d_model)
        _normal_(self.w1t, s, generator)
        _normal_(self.w2t, s, generator)
        with torch.no_grad():
            self.b1.zero_()
            self.b2.zero_()

    def load_reference(self, experts) -> "RoutedExperts":
        dev = self.w1t.device
        with torch.no_grad():
            for i, e in enumerate(experts):
                self.w1t[i].copy_(_as_tensor(np.asarray(e.w1).T, dev, self.w1t.dtype))
                self.b1[i].copy_(_as_tensor(np.asarray(e.b1).reshape(-1), dev, torch.float32))
                self.w2t[i].copy_(_as_tensor(np.asarray(e.w2).T, dev, self.w2t.dtype))
                self.b2[i].copy_(_as_tensor(np.asarray(e.b2).reshape(-1), dev, torch.float32))
        return self

    def forward(self, buf: torch.Tensor, group_rows: torch.Tensor, rows_clip: int,
                hidden: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                stream=None) -> torch.Tensor:
        """buf (G, C, d) with G a multiple of n_experts (EP receive buffers
        are (ranks * local experts)); group g uses expert g % n_experts."""
        return K.expert_ffn(buf, self.w1t, self.b1, self.w2t, self.b2, group_rows=group_rows,
                            rows_clip=rows_clip, hidden=hidden, out=out, stream=stream)


# ---------------------------------------------------------------------------
# layers


class _RoutedMoE(nn.Module):
    """Shared machinery of routed_moe (arch.py:463-486): gate -> dispatch ->
    grouped expert FFN -> (combine in the subclass).  With `ep_group` set the
    experts are sharded over the group's ranks and the dispatch / combine
    buffers travel through all-to-all (paper_2404_05019_b200.ep)."""

    def __init__(self, d_model, d_hidden, n_experts, k_routed, capacity_factor, noise_enabled,
                 dtype, device, generator, ep_group):
        super().__init__()
        if dtype not in (torch.bfloat16, torch.float32):
            raise ConfigError(f"dtype must be bf16 or fp32, got {dtype}")
        self.d_model, self.d_hidden, self.n_experts = d_model, d_hidden, n_experts
        self.k_routed, self.dtype = k_routed, dtype
        self.capacity = CapacityConfig(capacity_factor)
        self.gate = Top1Gate(d_model, n_experts, k=k_routed, noise_enabled=noise_enabled,
                             capacity_factor=capacity_factor, device=device, generator=generator)
        self.ep_group = ep_group
        ws = 1
        if ep_group is not None:
            import torch.distributed as dist
            ws = dist.get_world_size(ep_group)
            if n_experts % ws:
                raise ConfigError(f"n_experts={n_experts} not divisible by EP size {ws}")
        self.ep_size = ws
        self.experts = RoutedExperts(n_experts // ws, d_model, d_hidden, dtype, device, generator)
        # expert-parallel exchange: "nccl" (all-to-all of the capacity
        # buffers, ep.py) or "p2p" (our peer-memory kernels, ep_p2p.py)
        self.ep_backend = "nccl"
        self._xchg = None

    @property
    def noise_enabled(self):
        return self.gate.noise_enabled

    def ep_rank(self) -> int:
        if self.ep_group is None:
            return 0
        import torch.distributed as dist
        return dist.get_rank(self.ep_group)

    def _load_reference_common(self, layer):
        dev = self.gate.w_gate_t.device
        with torch.no_grad():
            self.gate.w_gate_t.copy_(_as_tensor(np.asarray(layer.gate.w_gate).T, dev, torch.float32))
            self.gate.w_noise_t.copy_(_as_tensor(np.asarray(layer.gate.w_noise).T, dev, torch.float32))
        el = self.experts.n_experts
        r = self.ep_rank()
        self.experts.load_reference(list(layer.experts)[r * el:(r + 1) * el])

    def route(self, x_src, eps=None, replay=None, generator=None, stream=None) -> GateDecision:
        if self.ep_group is not None:
            self._check_even_tokens(x_src.shape[0])
        dec = self.gate(x_src, eps=eps, generator=generator, replay=replay, stream=stream)
        if self.ep_group is not None and replay is not None and replay.indices is not None:
            dec = _agree_capacity(dec, self.ep_group)
        return dec

    def _check_even_tokens(self, t: int) -> None:
        """The exchanges move equal-split (E, C, d) blocks, C = ceil(cf*T*k/E)
        from each rank's own T (gating.py:134-135): every rank must route the
        same token count.  Checked once per new T (one small collective)."""
        seen = getattr(self, "_even_t", None)
        if seen == t:
            return
        import torch.distributed as dist
        ts = [None] * dist.get_world_size(self.ep_group)
        dist.all_gather_object(ts, t, group=self.ep_group)
        if len(set(ts)) != 1:
            raise ValueError(f"expert parallelism needs the same token count on every rank, "
                             f"got {ts}")
        self._even_t = t

    def routed_experts(self, x_src: torch.Tensor, dec: GateDecision, stream=None) -> torch.Tensor:
        """dispatch + expert FFN (+ EP exchange); returns the (N, C, d) expert
        output buffer that combine gathers from."""
        if self.ep_group is not None and self.ep_backend == "p2p":
            return self._p2p_routed(x_src, dec, stream)
        buf = K.dispatch(x_src, dec.indices, dec.slots, self.n_experts, dec.capacity, stream=stream)
        if self.ep_group is None:
            # rows(g) = min(pre-drop count, capacity) is computed in the kernel
            rows = dec.counts if dec.capacity == dec.quota else dec.kept_counts()
            return self.experts(buf, rows, dec.capacity, stream=stream)
        from . import ep
        return ep.expert_parallel_ffn(self.experts, buf, dec, self.ep_group)

    def peer_exchange(self, capacity: int, chunks: int = 1):
        """Peer-mapped buffers of the p2p backend (re-created when the
        per-chunk capacity, i.e. the per-rank token count, or the chunk count
        changes)."""
        from .ep_p2p import PeerExchange
        x = self._xchg
        if x is None or x.capacity != capacity or x.chunks != chunks:
            self._xchg = PeerExchange.from_group(self.ep_group, self.experts.n_experts, capacity,
                                                 self.d_model, self.dtype,
                                                 self.gate.w_gate_t.device, chunks=chunks)
        return self._xchg

    def _p2p_routed(self, x_src, dec, stream=None) -> torch.Tensor:
        """Synchronous p2p EP on one stream: rows to their owners, owner FFN,
        rows back; returns the (E, C, d) buffer combine gathers from."""
        xg = self.peer_exchange(dec.capacity)
        xg.dispatch(x_src, dec.indices, dec.slots, dec.counts, stream=stream)
        xg.expert_ffn_to_peers(self.experts, stream=stream)     # return fused into GEMM2
        xg.wait(1, stream)
        return xg.back.view(-1, dec.capacity, self.d_model)

    # -- training (autograd through the K7 kernels) ---------------------------
    def training_path(self) -> bool:
        """True when a forward must record the autograd graph."""
        return torch.is_grad_enabled() and any(p.requires_grad for p in self.parameters())

    def routed_train(self, src: torch.Tensor, dec: GateDecision):
        """Differentiable gate weights / aux and expert output buffer."""
        from . import training as TR
        if self.dtype != torch.bfloat16:
            raise NotImplementedError("backward kernels are bf16 only (the fp32 path is a "
                                      "forward parity path)")
        kept = dec.kept_counts().to(torch.int32)
        w, aux = TR.gate_weights_aux(self.gate, src, dec)
        buf = TR.DispatchFn.apply(src, dec.indices, dec.slots, kept, self.n_experts, dec.capacity)
        e = self.experts
        if self.ep_group is None:
            y = TR.FFNFn.apply(buf, e.w1t, e.b1, e.w2t, e.b2, None, kept, dec.capacity)
        else:
            from . import ep
            recv_counts = ep.exchange_counts(kept, self.ep_group)
            recv = TR.ExchangeFn.apply(buf, self.ep_group)
            y_local = TR.FFNFn.apply(recv, e.w1t, e.b1, e.w2t, e.b2, None, recv_counts,
                                     dec.capacity)
            y = TR.ExchangeFn.apply(y_local, self.ep_group)
        return w, aux, y, kept


class ScMoELayer(_RoutedMoE):
    """The shortcut-connected MoE layer: combine(SE(x_cur), routed(src), x_cur)
    — arch.moe_shared (arch.py:496-504).  `routed_src` is the preceding-layer
    representation chosen by the shortcut position (pos1 h_mlp_prev, pos2
    h_mh_prev, pos3 h_in; arch.py:593-597); None means x_cur (the plain
    shared-expert MoE)."""

    def __init__(self, d_model: int, d_hidden: int, n_experts: int, k_routed: int = 1,
                 combine_mode: str = "direct_add", capacity_factor: float = 2.0,
                 noise_enabled: bool = False, dtype=torch.bfloat16, device=None,
                 generator: Optional[torch.Generator] = None, ep_group=None):
        super().__init__(d_model, d_hidden, n_experts, k_routed, capacity_factor, noise_enabled,
                         dtype, device, generator, ep_group)
        if combine_mode not in COMBINE_MODES:
            raise ConfigError(f"unknown combine mode {combine_mode!r}")
        self.combine_mode = combine_mode
        self.shared = SharedExpert(d_model, d_hidden, dtype, device, generator)
        dev = self.gate.w_gate_t.device
        rows = {"direct_add": 0, "cg1": 1, "cg2": 2}[combine_mode]
        if rows:
            self.w_cg = nn.Parameter(torch.empty(rows, d_model, device=dev), requires_grad=False)
            _normal_(self.w_cg, 1.0 / math.sqrt(d_model), generator)
        else:
            self.w_cg = None

    @classmethod
    def from_reference(cls, layer, capacity=None, dtype=torch.bfloat16, device=None, ep_group=None):
        """Build from a reference arch.MoELayer (+ gating.CapacityConfig)."""
        d, n = np.asarray(layer.gate.w_gate).shape
        h = np.asarray(layer.shared.w1).shape[1]
        mode = getattr(getattr(layer, "combine", None), "mode", None) or getattr(layer, "combine_mode", "direct_add")
        cf = capacity.capacity_factor if capacity is not None else 2.0
        m = cls(d, h, n, k_routed=layer.gate.k, combine_mode=mode, capacity_factor=cf,
                noise_enabled=bool(layer.gate.noise_enabled), dtype=dtype, device=device,
                ep_group=ep_group)
        m._load_reference_common(layer)
        m.shared.load_reference(layer.shared)
        w_cg = getattr(getattr(layer, "combine", None), "w_cg", None)
        if w_cg is None:
            w_cg = getattr(layer, "w_cg", None)
        if m.w_cg is not None:
            with torch.no_grad():
                m.w_cg.copy_(_as_tensor(np.asarray(w_cg), m.w_cg.device, torch.float32))
        return m

    def forward(self, x_cur: torch.Tensor, routed_src: Optional[torch.Tensor] = None,
                residual: Optional[torch.Tensor] = None, eps: Optional[torch.Tensor] = None,
                replay: Optional[MoEReplay] = None, generator=None):
        """(out, decision, aux): out = combine(SE(x_cur), routed(src), x_cur)
        (+ residual when given, fusing the block's `h_mh_cur + feed_out`)."""
        src = x_cur if routed_src is None else routed_src
        if src.shape != x_cur.shape:
            raise ValueError("routed_src and x_cur must have the same shape")
        if self.training_path():
            from . import training as TR
            with torch.no_grad():
                dec = self.route(src, eps=eps, replay=replay, generator=generator)
            w, aux, y, kept = self.routed_train(src, dec)
            sh = self.shared
            # out = combine(SE(x), ...) + x: the residual gradient goes into the
            # shared expert's data-gradient GEMM (no separate autograd add)
            link = {} if (residual is not None and residual is x_cur and x_cur.requires_grad) \
                else None
            se = TR.FFNFn.apply(x_cur, sh.w1t, sh.b1, sh.w2t, sh.b2, None, None, x_cur.shape[0],
                                link)
            out = TR.CombineFn.apply(y, se, w, x_cur, self.w_cg, residual, dec.indices, dec.slots,
                                     kept, dec.capacity, self.combine_mode, link)
            return out, dec, aux
        dec = self.route(src, eps=eps, replay=replay, generator=generator)
        y = self.routed_experts(src, dec)
        if self.shared.can_fuse_combine(x_cur, dec, self.combine_mode):
            out = self.shared.forward_combine(x_cur, y, dec, residual=residual)
            return out, dec, dec.aux_loss()
        se = self.shared(x_cur)
        out = K.combine(y, dec.indices, dec.slots, dec.weights, dec.capacity, se_out=se,
                        mode=self.combine_mode, x_cur=x_cur, w_cg=self.w_cg, residual=residual)
        return out, dec, dec.aux_loss()


class Top2MoELayer(_RoutedMoE):
    """Standard top-k MoE baseline (k=2): arch.moe_standard (arch.py:489-493)
    — routed mixture on x, no shared expert, 2-way renormalised weights,
    token-major capacity, dropped selections zeroed without renormalising."""

    def __init__(self, d_model: int, d_hidden: int, n_experts: int, k_routed: int = 2,
                 capacity_factor: float = 2.0, noise_enabled: bool = False,
                 dtype=torch.bfloat16, device=None, generator: Optional[torch.Generator] = None,
                 ep_group=None):
        super().__init__(d_model, d_hidden, n_experts, k_routed, capacity_factor, noise_enabled,
                         dtype, device, generator, ep_group)

    @classmethod
    def from_reference(cls, layer, capacity=None, k=None, dtype=torch.bfloat16, device=None,
                       ep_group=None):
        d, n = np.asarray(layer.gate.w_gate).shape
        h = np.asarray(layer.experts[0].w1).shape[1]
        cf = capacity.capacity_factor if capacity is not None else 2.0
        m = cls(d, h, n, k_routed=k or layer.gate.k, capacity_factor=cf,
                noise_enabled=bool(layer.gate.noise_enabled), dtype=dtype, device=device,
                ep_group=ep_group)
        m._load_reference_common(layer)
        return m

    def forward(self, x: torch.Tensor, residual: Optional[torch.Tensor] = None,
                eps: Optional[torch.Tensor] = None, replay: Optional[MoEReplay] = None,
                generator=None):
        if self.training_path():
            from . import training as TR
            with torch.no_grad():
                dec = self.route(x, eps=eps, replay=replay, generator=generator)
            w, aux, y, kept = self.routed_train(x, dec)
            out = TR.CombineFn.apply(y, None, w, None, None, residual, dec.indices, dec.slots,
                                     kept, dec.capacity, "direct_add")
            return out, dec, aux
        dec = self.route(x, eps=eps, replay=replay, generator=generator)
        y = self.routed_experts(x, dec)
        out = K.combine(y, dec.indices, dec.slots, dec.weights, dec.capacity, residual=residual)
        return out, dec, dec.aux_loss()


class DGMoELayer(_RoutedMoE):
    """Dual-gating MoE (paper App. A.2, Eq. 20): two top-1 gatings with the
    same gate, one over the preceding-layer representation and one over the
    current one; with `dgmoe_constraint` a token whose current pick equals its
    preceding pick takes the current runner-up (arch.py:447-460, 507-533).
    out = routed(x_cur; dec_cur) + routed(x_prev; dec_prev), aux from the
    current gating.  Both dispatches share one (2N, C, d) buffer, so the two
    expert passes are a single grouped GEMM over 2N groups."""

    def __init__(self, d_model: int, d_hidden: int, n_experts: int,
                 capacity_factor: float = 2.0, dgmoe_constraint: bool = True,
                 noise_enabled: bool = False, dtype=torch.bfloat16, device=None,
                 generator: Optional[torch.Generator] = None, ep_group=None):
        if n_experts < 2:
            raise ConfigError("dual gating needs at least 2 experts")
        super().__init__(d_model, d_hidden, n_experts, 1, capacity_factor, noise_enabled,
                         dtype, device, generator, ep_group)
        self.constraint = dgmoe_constraint

    @classmethod
    def from_reference(cls, layer, capacity=None, constraint: bool = True, dtype=torch.bfloat16,
                       device=None, ep_group=None):
        d, n = np.asarray(layer.gate.w_gate).shape
        h = np.asarray(layer.experts[0].w1).shape[1]
        cf = capacity.capacity_factor if capacity is not None else 2.0
        m = cls(d, h, n, capacity_factor=cf, dgmoe_constraint=constraint,
                noise_enabled=bool(layer.gate.noise_enabled), dtype=dtype, device=device,
                ep_group=ep_group)
        m._load_reference_common(layer)
        return m

    def route_dual(self, x_cur, x_prev, eps=None, eps_prev=None, replay=None, generator=None):
        """(dec_cur, dec_prev) — dual_routing (arch.py:447-460) or, with the
        replay's indices and indices_prev, the pinned decisions
        (arch.py:518-520).  Noise (arch.py:514-515): the replay's draws, the
        given ones, else fresh draws (preceding gating first, as the
        reference's rng order)."""
        g = self.gate
        if replay is not None:
            eps = replay.eps if replay.eps is not None else eps
            eps_prev = replay.eps_prev if replay.eps_prev is not None else eps_prev
        if g.noise_enabled:
            shape = (x_cur.shape[0], self.n_experts)
            if eps_prev is None:
                eps_prev = torch.randn(shape, device=x_cur.device, generator=generator)
            if eps is None:
                eps = torch.randn(shape, device=x_cur.device, generator=generator)
            eps = _as_tensor(eps, x_cur.device, torch.float32)
            eps_prev = _as_tensor(eps_prev, x_cur.device, torch.float32)
        else:
            eps = eps_prev = None
        pinned = (replay is not None and replay.indices is not None
                  and replay.indices_prev is not None)
        if pinned:
            dec_prev = g(x_prev, eps=eps_prev, replay=MoEReplay(indices=replay.indices_prev,
                                                                dropped=replay.dropped_prev))
            dec_cur = g(x_cur, eps=eps, replay=MoEReplay(indices=replay.indices,
                                                         dropped=replay.dropped))
            return dec_cur, dec_prev
        dec_prev = g(x_prev, eps=eps_prev)
        quota = g.quota(x_cur.shape[0])
        excl = dec_prev.indices[:, 0] if self.constraint else None
        o = K.gate_topk(x_cur, g.w_gate_t, 1, quota,
                        w_noise_t=g.w_noise_t if g.noise_enabled else None,
                        eps=eps, exclude=excl)
        dec_cur = GateDecision(o.logits, o.indices, o.weights, o.dropped.bool(), o.slots, o.counts,
                               o.prob_sum, quota, quota, eps)
        return dec_cur, dec_prev

    def forward(self, x_cur: torch.Tensor, x_prev: torch.Tensor,
                residual: Optional[torch.Tensor] = None, eps=None, eps_prev=None,
                replay: Optional[MoEReplay] = None, generator=None):
        """(out, dec_cur, dec_prev, aux) — moe_dual_gating (arch.py:507-533)."""
        n = self.n_experts
        train = self.training_path()
        with torch.no_grad():
            dec_cur, dec_prev = self.route_dual(x_cur, x_prev, eps, eps_prev, replay, generator)
        # one (2N, cap, d) buffer for both dispatches
        cap = max(dec_cur.capacity, dec_prev.capacity)
        dec_cur, dec_prev = _with_capacity(dec_cur, cap), _with_capacity(dec_prev, cap)
        idx = torch.cat([dec_cur.indices, dec_prev.indices + n], dim=1).contiguous()
        slots = torch.cat([dec_cur.slots, dec_prev.slots], dim=1).contiguous()
        e = self.experts
        if train:
            if self.ep_group is not None:
                raise NotImplementedError("DGMoE training under expert parallelism")
            from . import training as TR
            w_cur, aux = TR.gate_weights_aux(self.gate, x_cur, dec_cur)
            kc, kp = dec_cur.kept_counts().int(), dec_prev.kept_counts().int()
            buf = torch.cat([TR.DispatchFn.apply(x_cur, dec_cur.indices, dec_cur.slots, kc, n, cap),
                             TR.DispatchFn.apply(x_prev, dec_prev.indices, dec_prev.slots, kp, n,
                                                 cap)])
            rows = torch.cat([kc, kp])
            y = TR.FFNFn.apply(buf, e.w1t, e.b1, e.w2t, e.b2, None, rows, cap)
            w = torch.cat([w_cur, dec_prev.weights], dim=1)
            out = TR.CombineFn.apply(y, None, w, None, None, residual, idx, slots,
                                     rows, cap, "direct_add")
            return out, dec_cur, dec_prev, aux
        if self.ep_group is not None:
            return self._forward_ep(x_cur, x_prev, dec_cur, dec_prev, cap, residual)
        buf = torch.empty(2 * n, cap, x_cur.shape[1], device=x_cur.device, dtype=x_cur.dtype)
        K.dispatch(x_cur, dec_cur.indices, dec_cur.slots, n, cap, out=buf[:n])
        K.dispatch(x_prev, dec_prev.indices, dec_prev.slots, n, cap, out=buf[n:])
        rows = torch.cat([dec_cur.kept_counts(), dec_prev.kept_counts()]).to(torch.int32)
        y = self.experts(buf, rows, cap)
        w = torch.cat([dec_cur.weights, dec_prev.weights], dim=1).contiguous()
        out = K.combine(y, idx, slots, w, cap, residual=residual)
        return out, dec_cur, dec_prev, dec_cur.aux_loss()

    def _forward_ep(self, x_cur, x_prev, dec_cur, dec_prev, cap, residual):
        """Expert parallelism (inference): the two gatings become ONE routing
        of 2T rows (x_cur then x_prev, top-1 each) over the N experts with
        2*cap slots per expert — the preceding gating's kept rows of expert e
        sit right after the current gating's (slot' = kept_cur[e] + slot), so
        every expert's rows stay contiguous — and go through the layer's EP
        exchange (NCCL or p2p) unchanged.  The combine gathers
        w_cur * y[e_cur, s_cur] + w_prev * y[e_prev, s'_prev] in the local
        path's selection order, so the result equals the local layer bit for
        bit (GEMM rows are independent of their position)."""
        self._check_even_tokens(x_cur.shape[0])
        n, cap2 = self.n_experts, 2 * cap
        kc = dec_cur.kept_counts().to(torch.int32)
        kp = dec_prev.kept_counts().to(torch.int32)
        s_cur, s_prev = dec_cur.slots, dec_prev.slots
        drop = torch.full_like(s_cur, cap2)
        slot_cur = torch.where(s_cur < cap, s_cur, drop)
        slot_prev = torch.where(s_prev < cap, kc[dec_prev.indices.long()] + s_prev, drop)
        idx2 = torch.cat([dec_cur.indices, dec_prev.indices]).contiguous()        # (2T, 1)
        slot2 = torch.cat([slot_cur, slot_prev]).contiguous()
        both = GateDecision(torch.cat([dec_cur.logits, dec_prev.logits]), idx2,
                            torch.cat([dec_cur.weights, dec_prev.weights]), slot2 >= cap2, slot2,
                            kc + kp, dec_cur.prob_sum, cap2, cap2)
        x2 = torch.cat([x_cur, x_prev])
        y = self.routed_experts(x2, both)                       # (N, 2 cap, d), global experts
        idx = torch.cat([dec_cur.indices, dec_prev.indices], dim=1).contiguous()
        slots = torch.cat([slot_cur, slot_prev], dim=1).contiguous()
        w = torch.cat([dec_cur.weights, dec_prev.weights], dim=1).contiguous()
        out = K.combine(y, idx, slots, w, cap2, residual=residual)
        return out, dec_cur, dec_prev, dec_cur.aux_loss()
