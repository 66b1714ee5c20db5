"""The ScMoE block pair (Block-MLP + Block-MoE) with scheduler-driven issue.

Wiring follows arch.model_forward's pair loop (arch.py:580-631):

    h_mh_prev  = h_in      + Attn_prev(feed(h_in))
    h_mlp_prev = h_mh_prev + MLP_prev(feed(h_mh_prev))
    h_mh_cur   = h_mlp_prev + Attn_cur(feed(h_mlp_prev))
    x_cur      = feed(h_mh_cur)                    (feed = LN iff pre_layernorm)
    out        = h_mh_cur + combine(SE(x_cur), routed(src), x_cur)
    src        = {pos1: h_mlp_prev, pos2: h_mh_prev, pos3: h_in}[pos]

The ops are issued in the order of the reference's shortcut-overlap DAG
(distsim.py:330-387): backbone pre-ops, gate + encode (dispatch kernel), the
window ops with the routed expert at the slot sched.choose_slot picks from
measured CUDA-event costs, then decode (combine kernel, fused with the
residual add).  Under expert parallelism the two all-to-alls run on a side
stream and overlap the window ops; `timeline.Recorder` captures every op on
its stream so the overlap fraction and exposed communication are measured on
the device.

Attention is the backbone, not the hot path: projections use the same
tcgen05 GEMM (bias-free), the core is torch SDPA.  `n_heads=1, seq_len=None,
causal=False` reproduces the reference's single-head unmasked attention over
all T rows with 1/sqrt(d_model) scaling (arch.py:354-358).
"""

from __future__ import annotations

import math
from typing import Dict, Optional

import torch
import torch.nn.functional as F
from torch import nn

from . import ep as ep_mod
from . import kernels as K
from . import sched
from .layers import (CapacityConfig, ConfigError, DGMoELayer, MoEReplay, ScMoELayer,
                     SharedExpert, Top2MoELayer, _as_tensor, _normal_)
from .timeline import Recorder

VARIANTS = ("scmoe", "shared", "standard", "dgmoe")
POSITIONS = ("pos1", "pos2", "pos3")


def layer_norm(x: torch.Tensor) -> torch.Tensor:
    """Parameter-free row LayerNorm, eps 1e-6 (arch.py:361-377)."""
    return F.layer_norm(x.float(), (x.shape[-1],), eps=1e-6).to(x.dtype)


# inference with the routed side stream: the shared expert's GEMM1 runs before
# the join, only its GEMM2 (with the fused combine) waits for the routed rows
SHARED_SPLIT_JOIN = True
PACKED_ATTENTION = True     # training attention through flash-attn's packed-QKV kernels
ATTN_TRAIN = "cudnn_packed"  # "cudnn_packed" | "flash_packed" | "autograd"
# windows of <= 192 rows (configs[1]: 144) run our own attention kernels on
# the packed QKV projection (csrc/attention.cu), training and inference
WINDOW_ATTENTION = True


class _WindowAttention(torch.autograd.Function):
    """Attention core on libscmoe's windowed kernels: reads the packed (T, 3d)
    QKV rows, returns O as (T, d) rows (the O projection's input), saves the
    row log-sum-exp; the backward writes dQKV straight into the packed
    layout.  No head permutes, no layout copies."""

    @staticmethod
    def forward(ctx, qkv, h, s, causal, scale):
        o, lse = K.window_attention_fwd(qkv, h, s, scale, causal)
        ctx.save_for_backward(qkv, o, lse)
        ctx.meta = (h, s, causal, scale)
        return o

    @staticmethod
    def backward(ctx, g):
        qkv, o, lse = ctx.saved_tensors
        h, s, causal, scale = ctx.meta
        dqkv = K.window_attention_bwd(qkv, o, g.contiguous(), lse, h, s, scale, causal)
        return dqkv, None, None, None, None


def _use_window_attention(qkv: torch.Tensor, s: int, hd: int) -> bool:
    return (WINDOW_ATTENTION and qkv.dtype == torch.bfloat16
            and K.window_attention_supported(s, hd))


class _CudnnPackedAttention(torch.autograd.Function):
    """Training attention core on cuDNN SDPA with the layouts under our
    control: q/k/v are views of the packed (T, 3d) projection, the output is
    returned as (T, d), and the backward writes dq/dk/dv straight into the
    packed (B, S, 3, H, hd) gradient with one copy per tensor (autograd's
    unbind/stack + permute copies were ~12% of the step).  The SDPA forward
    records its own small autograd graph (saved output / log-sum-exp), which
    the backward replays — no recomputation."""

    @staticmethod
    def forward(ctx, qkv, b, s, h, causal, scale):
        t, d3 = qkv.shape
        d = d3 // 3
        hd = d // h
        with torch.enable_grad():
            q5 = qkv.detach().view(b, s, 3, h, hd)
            q, k, v = (q5[:, :, i].transpose(1, 2).requires_grad_() for i in range(3))
            o = F.scaled_dot_product_attention(q, k, v, is_causal=causal, scale=scale)
        ctx.inner = (q, k, v, o)
        ctx.shape = (b, s, h, hd)
        if o.stride(1) == hd and o.stride(2) == h * hd:      # already (B, S, H, hd) in memory
            return o.detach().transpose(1, 2).reshape(t, d)
        return K.pack_heads([o.detach()]).view(t, d)

    @staticmethod
    def backward(ctx, g):
        q, k, v, o = ctx.inner
        b, s, h, hd = ctx.shape
        go = g.reshape(b, s, h, hd).transpose(1, 2)
        dq, dk, dv = torch.autograd.grad(o, (q, k, v), go)
        dqkv = K.pack_heads([dq, dk, dv])          # one vectorised pass into (B, S, 3, H, hd)
        ctx.inner = None
        return dqkv.view(b * s, 3 * h * hd), None, None, None, None, None


def _raise_if_nonfinite(loss: torch.Tensor) -> None:
    """grad.backward's divergence check (grad.py:84-85): FloatingPointError on
    a non-finite loss, before any parameter is updated."""
    if not bool(torch.isfinite(loss.detach()).all()):
        raise FloatingPointError("non-finite loss")


def _use_packed_attention(qkv: torch.Tensor, hd: int) -> bool:
    if not PACKED_ATTENTION or qkv.dtype != torch.bfloat16 or hd > 256 or hd % 8:
        return False
    try:
        import flash_attn  # noqa: F401
    except ImportError:
        return False
    return True


class Attention(nn.Module):
    """Multi-head SDPA with bias-free projections W_q, W_k, W_v, W_o (d x d)."""

    def __init__(self, d_model: int, n_heads: int = 1, seq_len: Optional[int] = None,
                 causal: bool = False, dtype=torch.bfloat16, device=None, generator=None):
        super().__init__()
        if d_model % n_heads:
            raise ConfigError("d_model must be divisible by n_heads")
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.d_model, self.n_heads, self.seq_len, self.causal = d_model, n_heads, seq_len, causal
        self.w_qkv_t = nn.Parameter(torch.empty(3 * d_model, d_model, device=dev, dtype=dtype), requires_grad=False)
        self.w_o_t = nn.Parameter(torch.empty(d_model, d_model, device=dev, dtype=dtype), requires_grad=False)
        _normal_(self.w_qkv_t, 1.0 / math.sqrt(d_model), generator)
        _normal_(self.w_o_t, 1.0 / math.sqrt(d_model), generator)

    def load_reference(self, a) -> "Attention":
        import numpy as np
        d = self.d_model
        dev, dt = self.w_qkv_t.device, self.w_qkv_t.dtype
        with torch.no_grad():
            for i, w in enumerate((a.w_q, a.w_k, a.w_v)):
                self.w_qkv_t[i * d:(i + 1) * d].copy_(_as_tensor(np.asarray(w).T, dev, dt))
            self.w_o_t.copy_(_as_tensor(np.asarray(a.w_o).T, dev, dt))
        return self

    def forward(self, x: torch.Tensor, residual: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Attention output (+ residual, fused into the W_o GEMM epilogue)."""
        t, d = x.shape
        h = self.n_heads
        s = self.seq_len or t
        if t % s:
            raise ValueError(f"{t} tokens do not split into sequences of {s}")
        b, hd = t // s, d // h
        train = torch.is_grad_enabled() and (self.w_qkv_t.requires_grad or x.requires_grad)
        # out = O(attn(QKV(x))) + x: the residual gradient is added in QKV's
        # data-gradient GEMM (LinearFn link) when x needs a gradient
        link = {} if (train and residual is x and x.requires_grad) else None
        if train:
            from .training import LinearFn
            qkv = LinearFn.apply(x, self.w_qkv_t, None, link)
        else:
            qkv = K.grouped_gemm(x, self.w_qkv_t, None)                    # (T, 3d)
        scale = 1.0 / math.sqrt(d) if h == 1 else 1.0 / math.sqrt(hd)
        if _use_window_attention(qkv, s, hd):
            if train:
                o = _WindowAttention.apply(qkv, h, s, self.causal, scale)
            else:
                o = K.window_attention_fwd(qkv, h, s, scale, self.causal, need_lse=False)[0]
        elif train and ATTN_TRAIN == "cudnn_packed" and qkv.dtype == torch.bfloat16:
            o = _CudnnPackedAttention.apply(qkv, b, s, h, self.causal, scale)
        elif train and ATTN_TRAIN == "flash_packed" and _use_packed_attention(qkv, hd):
            # training: flash-attn's packed-QKV kernels read (B, S, 3, H, hd) and
            # write dqkv in the same packed layout — no stack / permute copies
            # around the attention backward (they were ~12% of the step)
            from flash_attn import flash_attn_qkvpacked_func
            o = flash_attn_qkvpacked_func(qkv.view(b, s, 3, h, hd), causal=self.causal,
                                          softmax_scale=scale).reshape(t, d)
        else:
            q, k, v = qkv.view(b, s, 3, h, hd).permute(2, 0, 3, 1, 4).unbind(0)  # (B, H, S, hd)
            o = F.scaled_dot_product_attention(q, k, v, is_causal=self.causal, scale=scale)
            o = o.permute(0, 2, 1, 3).reshape(t, d).contiguous()
        if train:
            return LinearFn.apply(o, self.w_o_t, residual, link)
        return K.grouped_gemm(o, self.w_o_t, None, residual=residual)


class ScMoEBlockPair(nn.Module):
    """Block-MLP followed by a Block-MoE (ScMoE / shared-expert / top-k)."""

    _PAIR = True        # ScMoEBlock (every-block placement) drops the Block-MLP half

    def __init__(self, d_model: int, d_hidden: int, n_experts: int, variant: str = "scmoe",
                 shortcut_pos: Optional[str] = "pos2", k_routed: int = 1,
                 combine_mode: str = "direct_add", capacity_factor: float = 2.0,
                 noise_enabled: bool = False, pre_layernorm: bool = False, n_heads: int = 1,
                 seq_len: Optional[int] = None, causal: bool = False, dtype=torch.bfloat16,
                 device=None, generator=None, ep_group=None, dgmoe_constraint: bool = True,
                 chunks: int = 1, ep_backend: str = "nccl", p2p_ctas: int = 16,
                 p2p_return: str = "fused"):
        super().__init__()
        if chunks < 1:
            raise ConfigError("chunks must be >= 1")
        if ep_backend not in ("nccl", "p2p"):
            raise ConfigError(f"unknown ep_backend {ep_backend!r}")
        self.chunks = chunks
        # "nccl": all-to-all of the capacity buffers (ep.py); "p2p": our kernels
        # move only kept rows over peer memory (ep_p2p.py); p2p_ctas bounds the
        # side-stream copy kernels' grids so they run beside the window ops
        if p2p_return not in ("fused", "push"):
            raise ConfigError(f"unknown p2p_return {p2p_return!r}")
        # p2p return trip: "fused" — the owner's GEMM2 epilogue stores rows into
        # the sources' back buffers over peer memory, tile by tile; "push" — a
        # separate copy kernel on the comm stream after the FFN
        self.ep_backend, self.p2p_ctas, self.p2p_return = ep_backend, p2p_ctas, p2p_return
        # reserve p2p_ctas SMs for the exchange kernels during the window
        self.overlap_sm_budget = True
        # one GPU: the routed ops (gate, dispatch, expert FFN) on a side stream
        # beside the window ops — the shortcut makes them independent until
        # the shared expert's fused combine, so at N = 1 the two streams'
        # persistent GEMMs fill each other's wave tails (no exchange to hide).
        # Inference: on.  "decode" (default) joins at the combine: the shared
        # expert runs whole beside the routed path and the combine kernel
        # follows (shuffled graph A/B: faster than the fused shared-expert
        # combine in 4 of 5 runs, by 0.4-1.6%); True joins inside the shared
        # expert (GEMM1 before, GEMM2 with the fused combine after).
        # Training: routed_stream_train (experiment, slower)
        self.routed_stream_infer = "decode"
        self.routed_stream_train = False
        self._xchg = None
        if variant not in VARIANTS:
            raise ConfigError(f"unknown variant {variant!r}")
        if variant == "scmoe" and shortcut_pos not in POSITIONS:
            raise ConfigError(f"variant 'scmoe' needs shortcut_pos in {POSITIONS}")
        if variant != "scmoe":
            shortcut_pos = None
        if variant == "standard" and combine_mode != "direct_add":
            raise ConfigError("variant 'standard' has no shared/routed combination")
        self.variant, self.shortcut_pos = variant, shortcut_pos
        self.pre_layernorm = pre_layernorm
        self.dtype = dtype
        if not self._PAIR and variant == "scmoe" and shortcut_pos != "pos1":
            raise ConfigError("every-block shortcut placement supports pos1 only")  # arch.py:72-74
        kw = dict(dtype=dtype, device=device, generator=generator)
        if self._PAIR:
            self.attn_prev = Attention(d_model, n_heads, seq_len, causal, **kw)
            self.mlp_prev = SharedExpert(d_model, d_hidden, **kw)
        self.attn_cur = Attention(d_model, n_heads, seq_len, causal, **kw)
        if variant == "standard":
            self.moe = Top2MoELayer(d_model, d_hidden, n_experts, k_routed=k_routed,
                                    capacity_factor=capacity_factor, noise_enabled=noise_enabled,
                                    ep_group=ep_group, **kw)
        elif variant == "dgmoe":
            if not self._PAIR:
                raise ConfigError("dual gating is defined on block pairs only")  # arch.py:78-79
            self.moe = DGMoELayer(d_model, d_hidden, n_experts, capacity_factor=capacity_factor,
                                  dgmoe_constraint=dgmoe_constraint, noise_enabled=noise_enabled,
                                  ep_group=ep_group, **kw)
        else:
            self.moe = ScMoELayer(d_model, d_hidden, n_experts, k_routed=k_routed,
                                  combine_mode=combine_mode, capacity_factor=capacity_factor,
                                  noise_enabled=noise_enabled, ep_group=ep_group, **kw)
        self.ep_group = ep_group
        if hasattr(self.moe, "ep_backend"):
            self.moe.ep_backend = ep_backend
        self.offload = None
        self.offload_mode = "none"
        self.slot: Optional[int] = None
        self.last_costs: Optional[sched.CostVector] = None
        self._comm_stream: Optional[torch.cuda.Stream] = None

    # -- construction from the reference's parameter tree --------------------
    @classmethod
    def from_reference(cls, cfg, prev_blk, cur_blk, dtype=torch.bfloat16, device=None,
                       n_heads: int = 1, seq_len=None, causal=False, ep_group=None,
                       shortcut_pos: Optional[str] = None):
        """cfg: reference ModelConfig; prev_blk/cur_blk: BlockParams of one pair
        (prev_blk is ignored by the single-block ScMoEBlock)."""
        m = cls(cfg.d_model, cfg.d_hidden, cfg.n_experts, variant=cfg.variant,
                shortcut_pos=shortcut_pos or cfg.shortcut_pos, k_routed=cfg.k_routed,
                combine_mode=cfg.combine_mode, capacity_factor=cfg.capacity_factor,
                noise_enabled=cfg.noise_enabled, pre_layernorm=cfg.pre_layernorm,
                n_heads=n_heads, seq_len=seq_len, causal=causal, dtype=dtype, device=device,
                ep_group=ep_group, dgmoe_constraint=getattr(cfg, "dgmoe_constraint", True))
        if cls._PAIR:
            m.attn_prev.load_reference(prev_blk.attn)
            m.mlp_prev.load_reference(prev_blk.feed)
        m.attn_cur.load_reference(cur_blk.attn)
        cap = CapacityConfig(cfg.capacity_factor)
        layer = cur_blk.feed
        if cfg.variant == "standard":
            ref = Top2MoELayer.from_reference(layer, cap, k=cfg.k_routed, dtype=dtype,
                                              device=device, ep_group=ep_group)
        elif cfg.variant == "dgmoe":
            ref = DGMoELayer.from_reference(layer, cap, constraint=m.moe.constraint, dtype=dtype,
                                            device=device, ep_group=ep_group)
        else:
            ref = ScMoELayer.from_reference(layer, cap, dtype=dtype, device=device,
                                            ep_group=ep_group)
        m.moe = ref
        return m

    def _feed(self, h):
        return layer_norm(h) if self.pre_layernorm else h

    def peer_exchange(self, capacity: int, chunks: int = 1):
        """Peer-mapped buffers of the p2p backend — the MoE layer's own (one
        set per layer, re-created when the per-rank capacity or the chunk
        count changes)."""
        self._xchg = self.moe.peer_exchange(capacity, chunks)
        return self._xchg

    def _window_sm_budget(self) -> int:
        """SMs left to the window GEMMs while an exchange is in flight (0:
        all, when overlap_sm_budget is off)."""
        if not self.overlap_sm_budget:
            return 0
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        return max(2, sms - max(self.p2p_ctas, 2))

    def comm_stream(self) -> torch.cuda.Stream:
        if self._comm_stream is None:
            self._comm_stream = torch.cuda.Stream(priority=-1)
        return self._comm_stream

    def order(self):
        if self.variant == "dgmoe":
            return ["attn_prev", "mlp_prev", "attn_cur", "dual"]
        if self.variant == "scmoe":
            slot = self.slot
            if slot is None:
                # async expert offload: the expert after the whole window, so
                # the migration started at the gate point has the window to
                # hide behind (offload.py overlap_window); otherwise slot 0
                async_off = self.offload is not None and self.offload_mode == "async"
                slot = len(sched.WINDOW_OPS[self.shortcut_pos]) if async_off else 0
            o = sched.issue_order(self.shortcut_pos, slot)
        else:
            o = sched.sequential_order()
            if self.variant == "standard":
                o.remove("shared")
        if not self._PAIR:
            o = [n for n in o if n not in ("attn_prev", "mlp_prev")]
        return o

    # -- forward -------------------------------------------------------------
    def forward(self, h_in: torch.Tensor, eps=None, replay: Optional[MoEReplay] = None,
                recorder: Optional[Recorder] = None, return_taps: bool = False):
        """Returns (out, decision, aux[, taps])."""
        moe = self.moe
        rec = recorder or Recorder(enabled=False)
        st = torch.cuda.current_stream()
        use_ep = self.ep_group is not None
        cs = self.comm_stream() if use_ep else None
        env: Dict[str, object] = {}
        rec.begin(st)

        # residual adds are fused into the GEMM epilogues (arch.py:542, 587-589)
        def attn_prev():
            env["h_mh_prev"] = self.attn_prev(self._feed(h_in), residual=h_in)

        def mlp_prev():
            h = env["h_mh_prev"]
            env["h_mlp_prev"] = self.mlp_prev(self._feed(h), residual=h)

        def attn_cur():
            h = env["h_mlp_prev"]
            hc = self.attn_cur(self._feed(h), residual=h)
            env["h_mh_cur"] = hc
            env["x_cur"] = self._feed(hc)

        def src():
            if self.variant == "scmoe":
                return env[{"pos1": "h_mlp_prev", "pos2": "h_mh_prev", "pos3": "h_in"}[self.shortcut_pos]]
            return env["x_cur"]

        env["h_in"] = h_in
        if not self._PAIR:
            # every-block: the block input plays the preceding block's output
            # (src = h_in, arch.py:640) and attention reads it directly
            env["h_mh_prev"] = env["h_mlp_prev"] = h_in
        train = moe.training_path()
        if train:
            from . import training as TR
        # chunked pipelining (standard_pipeline / scmoe_overlap_pipeline,
        # distsim.py:277-300, 358-364): forward only
        chunks = self.chunks if not train else 1
        off = self.offload if not train else None
        if off is not None and (use_ep or chunks > 1):
            raise NotImplementedError("expert offload is a single-GPU, unchunked inference mode")
        p2p = use_ep and self.ep_backend == "p2p" and not train

        def gate():
            if train:
                with torch.no_grad():
                    dec = moe.route(src(), eps=eps, replay=replay)
                env["dec"] = dec
                env["kept"] = dec.kept_counts().to(torch.int32)
                env["w"], env["aux"] = TR.gate_weights_aux(moe.gate, src(), dec)
            else:
                env["dec"] = moe.route(src(), eps=eps, replay=replay)
                if chunks > 1:
                    env["cr"] = ep_mod.chunk_routing(env["dec"], chunks)
                if off is not None:
                    # activated experts -> device slots; the async migration
                    # starts at the (shortcut) gate point: issued once the
                    # next op is queued (the copy engine's host readback of
                    # the expert list then never idles the GPU)
                    env["plan"] = off.plan(env["dec"])
                    env["mig_pending"] = self.offload_mode == "async"

        def encode_offload():
            dec, plan = env["dec"], env["plan"]
            env["buf"] = K.dispatch(src(), plan.slot_idx, dec.slots, plan.n_slots, dec.capacity)

        def start_migration():
            env["bufs"], env["mig_ev"] = off.migrate_async(env["plan"])
            env["mig_pending"] = False

        def expert_offload():
            dec, plan = env["dec"], env["plan"]
            if env.get("mig_pending"):     # no window op between the gate and the expert
                start_migration()
            if self.offload_mode == "async":
                st.wait_event(env["mig_ev"])
                bufs = env["bufs"]
            else:
                bufs = off.migrate(plan)
            env["y"] = off.ffn(env["buf"], plan, bufs, dec.capacity)

        def encode_chunked():
            idx2, slot2, cc, rows = env["cr"]
            if p2p:
                # chunk c's kept rows straight to their owners, one p2p
                # exchange per chunk (own flags / epoch): the owner starts
                # chunk c's expert while chunk c+1 is still in flight
                dec = env["dec"]
                xg = self.peer_exchange(cc, chunks)
                sl = ep_mod.chunk_slots(dec, chunks, cc)
                cs.wait_stream(st)
                env["disp_evs"] = []
                for c in range(chunks):
                    with rec.op(f"dispatch{c}", "comm", cs):
                        xg.dispatch(src(), dec.indices, sl[c], rows[c], max_ctas=self.p2p_ctas,
                                    stream=cs, chunk=c)
                        ev = torch.cuda.Event()
                        ev.record(cs)
                    env["disp_evs"].append(ev)
                sl.record_stream(cs)
                rows.record_stream(cs)
                return
            # chunk-major buffer (chunks, E, Cc, d): chunk c's exchange is contiguous
            buf = K.dispatch(src(), idx2, slot2, chunks * moe.n_experts, cc)
            env["buf"] = buf.view(chunks, moe.n_experts, cc, -1)
            if use_ep:
                cs.wait_stream(st)
                env["pending"] = []
                for c in range(chunks):
                    with rec.op(f"dispatch{c}", "comm", cs):
                        env["pending"].append(ep_mod.dispatch_exchange(
                            env["buf"][c], rows[c].contiguous(), cc, self.ep_group, cs))

        def expert_chunked():
            idx2, slot2, cc, rows = env["cr"]
            if p2p:
                xg = self._xchg
                for c in range(chunks):
                    st.wait_event(env["disp_evs"][c])
                    if self.p2p_return == "fused":
                        xg.expert_ffn_to_peers(moe.experts, stream=st, chunk=c)
                    else:
                        xg.expert_ffn(moe.experts, signal=False, stream=st, chunk=c)
                        cs.wait_stream(st)
                        with rec.op(f"combine{c}", "comm", cs):
                            xg.push_back(max_ctas=self.p2p_ctas, stream=cs, chunk=c)
                            ev = torch.cuda.Event()
                            ev.record(cs)
                        env.setdefault("y_evs", []).append(ev)
                return
            y = torch.empty_like(env["buf"])
            evs = []
            for c in range(chunks):
                if use_ep:
                    p = env["pending"][c]
                    st.wait_event(p.event)
                    yc = moe.experts(p.recv, p.recv_counts, cc)
                    cs.wait_stream(st)
                    with rec.op(f"combine{c}", "comm", cs):
                        _, ev = ep_mod.combine_exchange(yc, self.ep_group, cs, out=y[c])
                    evs.append(ev)
                else:
                    moe.experts(env["buf"][c], rows[c].contiguous(), cc, out=y[c])
            env["y"] = y.view(chunks * moe.n_experts, cc, -1)
            env["y_evs"] = evs

        def decode_chunked():
            dec = env["dec"]
            idx2, slot2, cc, rows = env["cr"]
            if p2p:
                # every chunk's rows are back in the chunk-major back buffer
                for ev in env.get("y_evs", []):      # push form: join the comm stream
                    st.wait_event(ev)
                kw = dict(residual=env["h_mh_cur"], stream=st)
                if self.variant != "standard":
                    kw.update(se_out=env["se"], mode=moe.combine_mode, x_cur=env["x_cur"],
                              w_cg=moe.w_cg)
                env["out"] = self._xchg.combine_local(idx2, slot2, dec.weights, **kw)
                return
            for ev in env.get("y_evs", []):
                st.wait_event(ev)
            if self.variant == "standard":
                env["out"] = K.combine(env["y"], idx2, slot2, dec.weights, cc,
                                       residual=env["h_mh_cur"])
            else:
                env["out"] = K.combine(env["y"], idx2, slot2, dec.weights, cc, se_out=env["se"],
                                       mode=moe.combine_mode, x_cur=env["x_cur"], w_cg=moe.w_cg,
                                       residual=env["h_mh_cur"])

        def encode():
            dec = env["dec"]
            if chunks > 1:
                return encode_chunked()
            if off is not None:
                return encode_offload()
            if train:
                buf = TR.DispatchFn.apply(src(), dec.indices, dec.slots, env["kept"], moe.n_experts,
                                          dec.capacity)
                env["buf"] = buf
                if use_ep:
                    # the exchange runs on the comm stream beside the window ops;
                    # autograd runs its backward (the reverse exchange) on that
                    # stream too and synchronises the gradients across streams
                    cs.wait_stream(st)
                    buf.record_stream(cs)
                    with rec.op("dispatch", "comm", cs), torch.cuda.stream(cs):
                        env["recv_counts"] = ep_mod.exchange_counts(env["kept"], self.ep_group)
                        env["buf"] = TR.ExchangeFn.apply(buf, self.ep_group)
                        ev = torch.cuda.Event()
                        ev.record(cs)
                    env["disp_ev"] = ev
                return
            if p2p:
                # kept rows go straight to their owners over peer memory, on the
                # side stream beside the window ops (bounded grid)
                xg = self.peer_exchange(dec.capacity)
                cs.wait_stream(st)
                with rec.op("dispatch", "comm", cs):
                    xg.dispatch(src(), dec.indices, dec.slots, dec.counts, max_ctas=self.p2p_ctas,
                                stream=cs)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                env["disp_ev"] = ev
                return
            buf = K.dispatch(src(), dec.indices, dec.slots, moe.n_experts, dec.capacity)
            env["buf"] = buf
            if use_ep:
                cs.wait_stream(st)    # the span starts once the buffer is ready
                with rec.op("dispatch", "comm", cs):
                    env["pending"] = ep_mod.dispatch_exchange(buf, dec.kept_counts(), dec.capacity,
                                                              self.ep_group, cs)

        def expert():
            dec = env["dec"]
            if chunks > 1:
                return expert_chunked()
            if off is not None:
                return expert_offload()
            if train:
                e = moe.experts
                if use_ep:
                    st.wait_event(env["disp_ev"])
                    env["buf"].record_stream(st)
                    env["recv_counts"].record_stream(st)
                rows = env["recv_counts"] if use_ep else env["kept"]
                y = TR.FFNFn.apply(env["buf"], e.w1t, e.b1, e.w2t, e.b2, None, rows, dec.capacity)
                if not use_ep:
                    env["y"] = y
                    return
                cs.wait_stream(st)
                y.record_stream(cs)
                with rec.op("combine", "comm", cs), torch.cuda.stream(cs):
                    env["y"] = TR.ExchangeFn.apply(y, self.ep_group)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                env["y_ev"] = ev
                return
            if p2p:
                xg = self._xchg
                st.wait_event(env["disp_ev"])
                if self.p2p_return == "fused":
                    xg.expert_ffn_to_peers(moe.experts, stream=st)
                    env["y_ev"] = None
                    return
                xg.expert_ffn(moe.experts, signal=False, stream=st)
                cs.wait_stream(st)
                with rec.op("combine", "comm", cs):
                    xg.push_back(max_ctas=self.p2p_ctas, stream=cs)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                env["y_ev"] = ev
                return
            if use_ep:
                p = env["pending"]
                st.wait_event(p.event)
                y = moe.experts(p.recv, p.recv_counts, p.capacity)
                cs.wait_stream(st)
                with rec.op("combine", "comm", cs):
                    env["y"], env["y_ev"] = ep_mod.combine_exchange(y, self.ep_group, cs)
            else:
                rows = dec.counts if dec.capacity == dec.quota else dec.kept_counts()
                env["y"] = moe.experts(env["buf"], rows, dec.capacity)

        def shared():
            dec = env.get("dec")
            join = env.pop("join", None)     # routed side stream still running
            if ("y" in env and not train and not use_ep and chunks == 1 and off is None
                    and not env.get("no_fuse")
                    and self.variant in ("scmoe", "shared")
                    and moe.shared.can_fuse_combine(env["x_cur"], dec, moe.combine_mode)):
                # the routed rows are ready: the combine (+ the block residual)
                # runs in the shared expert's GEMM2 epilogue; decode is a no-op
                if join is not None:
                    # GEMM1 beside the routed expert; only GEMM2 waits for its rows
                    hid = moe.shared.hidden(env["x_cur"])
                    join()
                    env["out"] = moe.shared.combine_from_hidden(hid, env["y"], dec,
                                                                residual=env["h_mh_cur"])
                else:
                    env["out"] = moe.shared.forward_combine(env["x_cur"], env["y"], dec,
                                                            residual=env["h_mh_cur"])
                env["fused"] = True
                return
            if join is not None:
                join()
            # training: the block residual's gradient (combine) is added in the
            # shared expert's data-gradient GEMM when x_cur is the residual
            xc = env["x_cur"]
            env["link"] = {} if (train and xc is env.get("h_mh_cur") and xc.requires_grad) else None
            env["se"] = moe.shared(xc, link=env["link"])

        def decode():
            dec = env["dec"]
            if env.get("fused"):
                return
            if chunks > 1:
                return decode_chunked()
            if train:
                std = self.variant == "standard"
                if use_ep:
                    st.wait_event(env["y_ev"])
                    env["y"].record_stream(st)
                env["out"] = TR.CombineFn.apply(
                    env["y"], None if std else env["se"], env["w"], None if std else env["x_cur"],
                    None if std else moe.w_cg, env["h_mh_cur"], dec.indices, dec.slots, env["kept"],
                    dec.capacity, "direct_add" if std else moe.combine_mode,
                    None if std else env.get("link"))
                return
            if use_ep and env.get("y_ev") is not None:
                st.wait_event(env["y_ev"])
            if p2p:
                xg = self._xchg
                kw = dict(residual=env["h_mh_cur"], stream=st)
                if self.variant != "standard":
                    kw.update(se_out=env["se"], mode=moe.combine_mode, x_cur=env["x_cur"],
                              w_cg=moe.w_cg)
                env["out"] = xg.combine_local(dec.indices, dec.slots, dec.weights, **kw)
                return
            cidx = env["plan"].slot_idx if off is not None else dec.indices
            if self.variant == "standard":
                env["out"] = K.combine(env["y"], cidx, dec.slots, dec.weights, dec.capacity,
                                       residual=env["h_mh_cur"])
            else:
                env["out"] = K.combine(env["y"], cidx, dec.slots, dec.weights, dec.capacity,
                                       se_out=env["se"], mode=moe.combine_mode, x_cur=env["x_cur"],
                                       w_cg=moe.w_cg, residual=env["h_mh_cur"])

        def dual():
            # DGMoE: preceding gating on h_mh_prev, current on x_cur (arch.py:606-609)
            # eps = the current gating's noise; the preceding one comes from
            # the replay (eps_prev) or is drawn (arch.py:514-515)
            out, dc, dp, aux = moe(env["x_cur"], env["h_mh_prev"], residual=env["h_mh_cur"],
                                   eps=eps, replay=replay)
            env["out"], env["dec"], env["aux"] = out, (dc, dp), aux

        ops = dict(attn_prev=attn_prev, mlp_prev=mlp_prev, attn_cur=attn_cur, gate=gate,
                   encode=encode, expert=expert, shared=shared, decode=decode, dual=dual)
        # while an exchange kernel is in flight on the comm stream (dispatch:
        # from encode to the expert; push-form return: from the expert to
        # decode), the window ops' persistent GEMMs leave p2p_ctas SMs free so
        # the exchange runs concurrently instead of queueing behind them
        budget = self._window_sm_budget() if (use_ep and not train and (chunks == 1 or p2p)) else 0
        in_flight = False
        order = self.order()
        # (a per-op recorder — calibration, op timings — gets the serial order:
        # its events time each op alone)
        if ((self.routed_stream_train if train else self.routed_stream_infer) and not use_ep
                and chunks == 1 and off is None and self.variant == "scmoe" and recorder is None):
            side = self.comm_stream()
            forked = False
            join_at = ("decode",) if self.routed_stream_infer == "decode" else ("shared", "decode")
            if self.routed_stream_infer == "decode":
                env["no_fuse"] = True
            for name in order:
                if name in ("gate", "encode", "expert"):
                    if not forked:
                        side.wait_stream(st)
                        forked = True
                    with rec.op(name, "compute", side), torch.cuda.stream(side):
                        ops[name]()
                    continue
                if name in join_at and forked:
                    forked = False

                    def _join():
                        st.wait_stream(side)      # the combine reads the routed rows
                        for key in ("y", "buf", "w", "aux", "kept"):
                            t = env.get(key)
                            if isinstance(t, torch.Tensor):
                                t.record_stream(st)
                        dec = env["dec"]
                        for t in (dec.logits, dec.indices, dec.weights, dec.dropped, dec.slots,
                                  dec.counts, dec.prob_sum):
                            t.record_stream(st)
                    if name == "shared" and SHARED_SPLIT_JOIN:
                        env["join"] = _join       # shared() joins between its two GEMMs
                    else:
                        _join()
                with rec.op(name, "compute", st):
                    ops[name]()
            order = []
        for name in order:
            if name == "expert":   # NCCL combine / push return run behind the expert
                in_flight = (not p2p) or self.p2p_return == "push"
            with rec.op(name, "compute", st):
                if in_flight and budget and name not in ("expert", "decode"):
                    with K.gemm_sm_budget(budget):
                        ops[name]()
                else:
                    ops[name]()
            if name == "encode":
                in_flight = True
            elif env.get("mig_pending") and name != "gate":
                start_migration()
        dec = env["dec"]
        if self.variant == "dgmoe":
            res = (env["out"], dec, env["aux"])       # decision = (current, preceding)
        else:
            res = (env["out"], dec, env["aux"] if train else dec.aux_loss())
        if return_taps:
            taps = {k: env[k] for k in ("h_mh_prev", "h_mlp_prev", "h_mh_cur", "x_cur")}
            taps["src"] = src()
            return res + (taps,)
        return res

    # -- memory-limited inference -----------------------------------------------
    def enable_offload(self, mode: str = "async", engine: str = "copy") -> "ScMoEBlockPair":
        """Move the routed experts to pinned host memory (offload.py).  "async"
        starts the migration at the gate point (needs the ScMoE shortcut
        routing to overlap anything), "blocking" right before the expert
        computation, "none" keeps them resident.  engine: "copy" (copy-engine
        transfers, the expert list read back to the host) or "sm" (gather
        kernel, no host round trip, graph-capturable)."""
        from .offload import ENGINES, MODES, ExpertOffload
        if mode not in MODES:
            raise ConfigError(f"unknown offload mode {mode!r}")
        if engine not in ENGINES:
            raise ConfigError(f"unknown migration engine {engine!r}")
        if mode == "none":
            return self
        if self.variant == "dgmoe" or self.ep_group is not None:
            raise ConfigError("expert offload supports single-GPU ScMoE / shared / top-k layers")
        if self.offload is None:
            self.offload = ExpertOffload(self.moe.experts, self.moe.k_routed, engine)
        self.offload.engine = engine
        self.offload_mode = mode
        return self

    # -- training ----------------------------------------------------------------
    def train_step(self, h_in: torch.Tensor, lr: float = 0.01, aux_coeff: float = 0.01,
                   target: Optional[torch.Tensor] = None, dp_group=None, update: bool = True,
                   check_finite: bool = False):
        """One optimisation step of the reference objective (grad.py:52-67):
        loss = mean(out) (or sum((out - target)^2) / T, LossSpec "mse") +
        aux_coeff * aux, backward through the K7 kernels, data-parallel
        all-reduce of the replicated parameters (N > 1), in-place SGD
        (grad.py:330-331).  Returns the loss (device tensor, no sync).
        check_finite: raise FloatingPointError("non-finite loss") before the
        update, as grad.backward does (grad.py:84-85) — one host sync."""
        from . import training as TR
        for p in self.parameters():
            p.grad = None
        out, dec, aux = self(h_in)
        if target is None:
            loss = TR.mean_loss(out)      # fp32 accumulation, no fp32 copy of out
        else:
            loss = (out.float() - target.float()).pow(2).sum() / out.shape[0]
        loss = loss + aux_coeff * aux
        loss.backward()
        if check_finite:
            _raise_if_nonfinite(loss)
        if dp_group is not None or self.ep_group is not None:
            TR.allreduce_replicated_grads(self, dp_group if dp_group is not None else self.ep_group,
                                          experts_sharded=self.ep_group is not None)
        if update:
            TR.sgd_step(self.parameters(), lr)
        return loss.detach()

    # -- adaptive scheduling ---------------------------------------------------
    def calibrate(self, h_in: torch.Tensor, repeats: int = 3) -> sched.ScheduleChoice:
        """Measure window-op, expert and all-to-all durations with CUDA events
        and pick the expert slot (Eq. 10) — the paper's adaptive operator
        scheduling, on real device timings."""
        if self.variant != "scmoe":
            raise ConfigError("only the ScMoE variant has an overlap window")
        durs: Dict[str, float] = {}
        for _ in range(repeats):
            rec = Recorder()
            self.forward(h_in, recorder=rec)
            for k, v in rec.durations().items():
                durs[k] = min(durs.get(k, float("inf")), v)
        window = [n for n in sched.WINDOW_OPS[self.shortcut_pos]
                  if self._PAIR or n not in ("attn_prev", "mlp_prev")]
        comm_d = durs.get("dispatch", 0.0)
        comm_c = durs.get("combine", 0.0)
        if (self.ep_group is not None and self.ep_backend == "p2p" and self.p2p_return == "fused"
                and comm_c == 0.0):
            # the fused return travels inside the expert's GEMM2 epilogue and
            # has no span of its own: measure the same transfer as the
            # push-form return kernel so Eq. 10 sees t_comb > 0
            self.p2p_return = "push"
            try:
                for _ in range(repeats):
                    rec = Recorder()
                    self.forward(h_in, recorder=rec)
                    d = rec.durations().get("combine", 0.0)
                    comm_c = d if comm_c == 0.0 else min(comm_c, d)
            finally:
                self.p2p_return = "fused"
        expert_ms = durs.get("expert", 0.0)
        if self.ep_group is not None:
            # the compute-stream "expert" span includes waiting on the
            # dispatch; the exchange itself is timed on the comm stream
            expert_ms = max(0.0, expert_ms - comm_d)
        cv = sched.CostVector([durs.get(n, 0.0) for n in window], comm_d, comm_c, expert_ms)
        choice = sched.choose_slot(cv)
        self.slot = choice.slot
        self.last_costs = cv
        return choice


class ScMoEBlock(ScMoEBlockPair):
    """One Transformer block whose feed is the MoE layer — the every-block
    placement (moe_frequency "every-block", arch.py:632-663):

        h_mh = h_in + Attn(feed(h_in));  out = h_mh + MoE(feed(h_mh), src)

    with src = h_in (ScMoE pos1, the previous block's output), else feed(h_mh).
    The gate and dispatch of the ScMoE variant only need h_in, so they are
    issued before the attention and the all-to-alls overlap attention + SE."""

    _PAIR = False

    def __init__(self, d_model: int, d_hidden: int, n_experts: int, variant: str = "scmoe",
                 shortcut_pos: Optional[str] = "pos1", **kw):
        super().__init__(d_model, d_hidden, n_experts, variant=variant,
                         shortcut_pos=shortcut_pos, **kw)


class ScMoEModel(nn.Module):
    """The reference's model (arch.model_forward, arch.py:553-665) on the GPU:
    n_blocks Transformer blocks with the MoE feed every second block (block
    pairs, ScMoEBlockPair) or every block (ScMoEBlock).  Constructor fields
    are ModelConfig's (arch.py:39-54); `first_layer_pos1` routes the first
    pair from pos1 (arch.py:594-595).  forward -> (out, decisions, auxes)."""

    def __init__(self, n_blocks: int, d_model: int, d_hidden: int, n_experts: int,
                 k_routed: int = 1, moe_frequency: str = "every-second-block",
                 variant: str = "standard", shortcut_pos: Optional[str] = None,
                 combine_mode: str = "direct_add", capacity_factor: float = 2.0,
                 noise_enabled: bool = False, first_layer_pos1: bool = False,
                 pre_layernorm: bool = False, n_heads: int = 1, seq_len: Optional[int] = None,
                 causal: bool = False, dtype=torch.bfloat16, device=None, generator=None,
                 ep_group=None, dgmoe_constraint: bool = True, _build: bool = True):
        super().__init__()
        if moe_frequency not in ("every-second-block", "every-block"):
            raise ConfigError(f"unknown moe_frequency {moe_frequency!r}")
        if moe_frequency == "every-second-block" and n_blocks % 2:
            raise ConfigError("every-second-block placement needs an even block count")
        if variant == "scmoe" and moe_frequency == "every-block" and shortcut_pos != "pos1":
            raise ConfigError("every-block shortcut placement supports pos1 only")
        self.moe_frequency, self.variant = moe_frequency, variant
        kw = dict(k_routed=k_routed, combine_mode=combine_mode, capacity_factor=capacity_factor,
                  noise_enabled=noise_enabled, pre_layernorm=pre_layernorm, n_heads=n_heads,
                  seq_len=seq_len, causal=causal, dtype=dtype, device=device,
                  generator=generator, ep_group=ep_group)
        if variant == "dgmoe":
            kw["dgmoe_constraint"] = dgmoe_constraint
        blocks = []
        if _build:
            if moe_frequency == "every-second-block":
                for pair in range(n_blocks // 2):
                    pos = shortcut_pos
                    if variant == "scmoe" and first_layer_pos1 and pair == 0:
                        pos = "pos1"
                    blocks.append(ScMoEBlockPair(d_model, d_hidden, n_experts, variant=variant,
                                                 shortcut_pos=pos, **kw))
            else:
                for _ in range(n_blocks):
                    blocks.append(ScMoEBlock(d_model, d_hidden, n_experts, variant=variant,
                                             shortcut_pos=shortcut_pos, **kw))
        self.blocks = nn.ModuleList(blocks)

    @classmethod
    def from_reference(cls, cfg, params, dtype=torch.bfloat16, device=None, n_heads: int = 1,
                       seq_len=None, causal=False, ep_group=None):
        """cfg: reference ModelConfig; params: ModelParams (arch.py:150-151)."""
        m = cls(cfg.n_blocks, cfg.d_model, cfg.d_hidden, cfg.n_experts, k_routed=cfg.k_routed,
                moe_frequency=cfg.moe_frequency, variant=cfg.variant,
                shortcut_pos=cfg.shortcut_pos, combine_mode=cfg.combine_mode,
                capacity_factor=cfg.capacity_factor, noise_enabled=cfg.noise_enabled,
                first_layer_pos1=cfg.first_layer_pos1, pre_layernorm=cfg.pre_layernorm,
                n_heads=n_heads, seq_len=seq_len, causal=causal, dtype=dtype, device=device,
                ep_group=ep_group, _build=False)
        kw = dict(dtype=dtype, device=device, n_heads=n_heads, seq_len=seq_len, causal=causal,
                  ep_group=ep_group)
        blocks = list(params.blocks)
        if cfg.moe_frequency == "every-second-block":
            for pair in range(cfg.n_blocks // 2):
                pos = "pos1" if (cfg.variant == "scmoe" and cfg.first_layer_pos1 and pair == 0) \
                    else None
                m.blocks.append(ScMoEBlockPair.from_reference(
                    cfg, blocks[2 * pair], blocks[2 * pair + 1], shortcut_pos=pos, **kw))
        else:
            for b in blocks:
                m.blocks.append(ScMoEBlock.from_reference(cfg, None, b, **kw))
        return m

    def forward(self, tokens: torch.Tensor, replay=None):
        h = tokens
        decs, auxes = [], []
        for i, blk in enumerate(self.blocks):
            h, dec, aux = blk(h, replay=None if replay is None else replay[i])
            decs.append(dec)
            auxes.append(aux)
        return h, decs, auxes

    def train_step(self, tokens: torch.Tensor, lr: float = 0.01, aux_coeff: float = 0.01,
                   target: Optional[torch.Tensor] = None, dp_group=None, update: bool = True,
                   check_finite: bool = False):
        """grad.compute_loss (mean / mse + aux_coeff * sum aux) + SGD;
        check_finite as in ScMoEBlockPair.train_step (grad.py:84-85)."""
        from . import training as TR
        for p in self.parameters():
            p.grad = None
        out, _, auxes = self(tokens)
        loss = TR.mean_loss(out) if target is None else \
            (out.float() - target.float()).pow(2).sum() / out.shape[0]
        for a in auxes:
            loss = loss + aux_coeff * a
        loss.backward()
        if check_finite:
            _raise_if_nonfinite(loss)
        ep = self.blocks[0].ep_group if len(self.blocks) else None
        if dp_group is not None or ep is not None:
            TR.allreduce_replicated_grads(self, dp_group if dp_group is not None else ep,
                                          experts_sharded=ep is not None)
        if update:
            TR.sgd_step(self.parameters(), lr)
        return loss.detach()
