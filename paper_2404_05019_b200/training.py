"""Training path (K7): autograd Functions whose forward AND backward run on
libscmoe kernels.

Semantics follow the reference's tape (scmoelab/tape.py, grad.py:52-86):
  * routing index sets and drop masks are constants (straight-through,
    tape.py:11-13);
  * the objective is loss + aux_coeff * sum(aux) (grad.py:52-67, aux_coeff 0.01
    by default, LossSpec grad.py:28-40), so the top-1 gate only receives
    gradient through the balance loss (arch.py:436-439) — its masked-softmax
    weight is identically 1;
  * GELU is the exact erf GELU (tape.py:137-142).

Kernels used in backward: the tcgen05 GEMM reading the stored K-major weights
transposed (MN-major operand) with the GELU-backward epilogue (dZ = dH *
gelu'(Z)), the split-K grouped weight-gradient GEMM, grouped column sums for
bias gradients, the scaled dispatch (combine backward) and the combine kernel
used as a gather-sum (dispatch backward).  Only the bf16 path has backward
kernels; the fp32 parity path is forward-only.
"""

from __future__ import annotations

from typing import Optional

import torch

from . import _lib
from . import kernels as K

_NK, _KN = _lib.W_NK, _lib.W_KN


def _as_param_grad(g: torch.Tensor, like: torch.Tensor) -> torch.Tensor:
    return g.to(like.dtype).view(like.shape)


def _park(link: dict, dy: torch.Tensor) -> None:
    """Park a residual gradient for the data-gradient GEMM of the Function
    that reads the same input (see LinearFn), tagged with the backward pass
    that produced it."""
    link["dy"] = (torch._C._current_graph_task_id(), dy)


def _take(link) -> Optional[torch.Tensor]:
    """The gradient parked in THIS backward pass, or None.  A stale entry
    (parked by a partial backward, e.g. autograd.grad w.r.t. one weight,
    whose consumer never ran) is dropped instead of being added twice."""
    if link is None:
        return None
    item = link.pop("dy", None)
    if item is None or item[0] != torch._C._current_graph_task_id():
        return None
    return item[1]


# Backward concurrency: a layer's data-gradient GEMM and its weight-gradient
# GEMM are independent.  With CONCURRENT_BWD the weight gradient runs on a
# side stream beside the data gradient, each persistent GEMM on half of the
# SMs (scmoe_set_gemm_sm_budget): every K = 384 GEMM of the configs[1] step
# carries a ~5-8 us fixed cost (pipeline fill, one-tile epilogue, teardown,
# scripts/wgrad_scaling.py) that the pair now pays side by side.
CONCURRENT_BWD = True
# SMs of the side (weight-gradient) / main (data-gradient) GEMMs while both
# run, as fractions of the device's SMs (0 = no budget)
# concurrent backward: db2 (column sums of dy) beside the dz GEMM with dW2,
# db1 beside the dx GEMM with dW1 — balances the two streams' phases
SPLIT_COLSUM = True
BWD_SIDE_FRAC = 0.5
BWD_MAIN_FRAC = 0.5
_SIDE = {}


class _Side:
    """Fork the current stream onto the device's side stream for `with`, with
    the GEMM SM budget halved for launches issued inside; join() makes the
    current stream wait for everything the side stream was given."""

    def __init__(self, dev: torch.device):
        self.main = torch.cuda.current_stream(dev)
        st = _SIDE.get(dev.index)
        if st is None:
            st = _SIDE[dev.index] = torch.cuda.Stream(dev)
        self.side = st
        n = torch.cuda.get_device_properties(dev).multi_processor_count
        self.side_sms = int(n * BWD_SIDE_FRAC)
        self.main_sms = int(n * BWD_MAIN_FRAC)
        self.outs = []

    def fork(self):
        self.side.wait_stream(self.main)

    def on_side(self):
        return torch.cuda.stream(self.side)

    def keep(self, *ts):
        self.outs.extend(t for t in ts if t is not None)

    def join(self):
        self.main.wait_stream(self.side)
        for t in self.outs:                 # produced on the side stream, consumed on main
            t.record_stream(self.main)


def _wgrad_dtype(w: torch.Tensor) -> torch.dtype:
    """bf16 weights get their gradient straight from the split reduction."""
    return torch.bfloat16 if w.dtype == torch.bfloat16 else torch.float32


class LinearFn(torch.autograd.Function):
    """y = x @ wt^T (+ residual); wt is (n_out, k_in) (bias-free projection).

    `link` (a dict shared by two LinearFns of one sub-block, or None) moves a
    residual gradient into a data-gradient GEMM: for h -> QKV ... -> O + h,
    the O projection (it has the residual) parks dy in the link instead of
    returning it, and the QKV projection (input h) adds it in its dx GEMM's
    residual epilogue — the same sum as autograd's add, one kernel fewer.
    Autograd runs the O projection's backward first (QKV's output feeds it)."""

    @staticmethod
    def forward(ctx, x, wt, residual, link=None):
        y = K.grouped_gemm(x, wt, None, residual=residual)
        ctx.save_for_backward(x, wt)
        ctx.has_res = residual is not None
        ctx.link = link
        return y

    @staticmethod
    def backward(ctx, dy):
        x, wt = ctx.saved_tensors
        dy = dy.contiguous()
        dx = dwt = None
        link = ctx.link
        if ctx.has_res and link is not None:       # the residual's gradient, parked
            _park(link, dy)
            res_grad = None
        else:
            res_grad = dy if ctx.has_res else None
        both = ctx.needs_input_grad[0] and ctx.needs_input_grad[1]
        sd = _Side(dy.device) if (CONCURRENT_BWD and both) else None
        if sd is not None:
            # dW on the side stream beside dx, half of the SMs each
            sd.fork()
            with K.gemm_sm_budget(sd.main_sms):
                with sd.on_side(), K.gemm_sm_budget(sd.side_sms):
                    dwt = _as_param_grad(K.grouped_wgrad(dy, x, out_dtype=_wgrad_dtype(wt)), wt)
                extra = _take(link) if not ctx.has_res else None
                dx = K.grouped_gemm_ex(dy, wt, _KN, wt.shape[1], residual=extra)
            sd.keep(dwt)
            sd.join()
            return dx, dwt, res_grad, None
        if ctx.needs_input_grad[0]:
            extra = _take(link) if not ctx.has_res else None
            dx = K.grouped_gemm_ex(dy, wt, _KN, wt.shape[1], residual=extra)
        if ctx.needs_input_grad[1]:
            dwt = _as_param_grad(K.grouped_wgrad(dy, x, out_dtype=_wgrad_dtype(wt)), wt)
        return dx, dwt, res_grad, None


# training FFN GELU: a separate full-occupancy forward pass that writes
# gelu(z) and gelu'(z) (True; the backward's data-gradient GEMM multiplies by
# gelu'(z) in its epilogue), or the GEMM epilogues evaluating erf (False); at
# d = 384 the K = 384 tiles make erf in the GEMM epilogues the bottleneck
# (csrc/gelu.cu)
SPLIT_GELU = True


def _wsum(per_group: torch.Tensor, n_wgroups: int) -> torch.Tensor:
    """(G, n) per-group sums -> (W, n): group g feeds weight group g % W."""
    g = per_group.shape[0]
    if g == n_wgroups:
        return per_group
    return per_group.view(g // n_wgroups, n_wgroups, -1).sum(0)


class FFNFn(torch.autograd.Function):
    """expert_forward (arch.py:349-351) over groups, + optional residual.

    x (G, C, d) or (T, d); w1t (W, h, d), b1 (W, h), w2t (W, d, h), b2 (W, d).
    Rows past rows(g) are zero-padded in the saved activations so the weight
    gradients can sum whole 64-row blocks."""

    @staticmethod
    def forward(ctx, x, w1t, b1, w2t, b2, residual, group_rows, rows_clip, link=None):
        two_d = x.dim() == 2
        x3 = x.unsqueeze(0) if two_d else x
        w13 = w1t.unsqueeze(0) if w1t.dim() == 2 else w1t
        w23 = w2t.unsqueeze(0) if w2t.dim() == 2 else w2t
        G, C, d = x3.shape
        h = w13.shape[1]
        if SPLIT_GELU:
            # plain bias GEMM -> z, then h = gelu(z) and gelu'(z) in one
            # full-occupancy pass (zero-padded tails for the weight
            # gradients); the backward multiplies by the saved gelu'(z) in
            # its data-gradient GEMM's epilogue
            z = K.grouped_gemm_ex(x3, w13, _NK, h, bias=b1.view(-1, h), epilogue=_lib.EPI_BIAS,
                                  group_rows=group_rows, rows_clip=rows_clip)
            hid, dgelu = K.gelu_fwd_grad(z, group_rows, rows_clip)
            z = dgelu
        else:
            z = torch.empty(G, C, h, device=x.device, dtype=x.dtype)
            hid = K.grouped_gemm_ex(x3, w13, _NK, h, bias=b1.view(-1, h), aux_out=z,
                                    epilogue=_lib.EPI_BIAS_GELU, group_rows=group_rows,
                                    rows_clip=rows_clip, zero_tail=group_rows is not None)
        res3 = None if residual is None else residual.view(G, C, d)
        y = K.grouped_gemm_ex(hid, w23, _NK, d, bias=b2.view(-1, d), residual=res3,
                              group_rows=group_rows, rows_clip=rows_clip)
        ctx.save_for_backward(x3, z, hid, w13, w23, group_rows)   # z: gelu'(z) when split
        ctx.meta = (two_d, rows_clip, residual is not None, b1.shape, b2.shape, w1t.shape,
                    w2t.shape)
        # y = FFN(x) + x (the Block-MLP): the data gradient adds dy in its
        # GEMM epilogue instead of a separate autograd add
        ctx.res_is_x = residual is x and group_rows is None
        # link: a residual gradient of x parked by a later Function (the
        # ScMoE combine), added here like LinearFn's link
        ctx.link = link if (group_rows is None and residual is None) else None
        return y.view(C, d) if two_d else y

    @staticmethod
    def backward(ctx, dy):
        x3, z, hid, w13, w23, group_rows = ctx.saved_tensors
        two_d, rows_clip, has_res, b1_shape, b2_shape, w1_shape, w2_shape = ctx.meta
        G, C, d = x3.shape
        W, h, _ = w13.shape
        dy3 = dy.contiguous().view(G, C, d)
        grouped = group_rows is not None
        if grouped:
            K.zero_tails(dy3, group_rows, rows_clip)
        epi = _lib.EPI_MUL_AUX if SPLIT_GELU else _lib.EPI_GELU_BWD
        fuse_res = has_res and ctx.res_is_x
        parked = _take(ctx.link)
        extra = dy3 if fuse_res else (parked.view(G, C, d) if parked is not None else None)
        sd = _Side(dy3.device) if CONCURRENT_BWD else None
        if sd is not None:
            sd.fork()
        with K.gemm_sm_budget(sd.main_sms if sd is not None else 0):
            if sd is not None:
                with sd.on_side(), K.gemm_sm_budget(sd.side_sms):   # dW2, db2 beside dz (read dy)
                    dw2t = K.grouped_wgrad(dy3, hid, n_wgroups=W, group_rows=group_rows,
                                           rows_clip=rows_clip, out_dtype=_wgrad_dtype(w23))
                    if SPLIT_COLSUM:
                        db2_g = K.grouped_colsum(dy3, group_rows, rows_clip)
            # SPLIT_GELU: z holds gelu'(z) (saved by the forward): dz = (dy W2) *
            # gelu'(z) in the data-gradient GEMM's epilogue, zero tails
            dz = K.grouped_gemm_ex(dy3, w23, _KN, h, aux_in=z, epilogue=epi,
                                   group_rows=group_rows, rows_clip=rows_clip, zero_tail=grouped)
            if sd is not None:
                sd.fork()                    # dz ready
                with sd.on_side(), K.gemm_sm_budget(sd.side_sms):   # dW1, bias grads beside dx
                    dw1t = K.grouped_wgrad(dz, x3, n_wgroups=W, group_rows=group_rows,
                                           rows_clip=rows_clip, out_dtype=_wgrad_dtype(w13))
                    if SPLIT_COLSUM:
                        db1_g = K.grouped_colsum(dz, group_rows, rows_clip)
                    else:
                        db2_g, db1_g = K.grouped_colsum2(dy3, dz, group_rows, rows_clip)
            dx = K.grouped_gemm_ex(dz, w13, _KN, d, group_rows=group_rows, rows_clip=rows_clip,
                                   residual=extra)
        if sd is not None:
            sd.keep(dw2t, dw1t, db2_g, db1_g)
            sd.join()
        else:
            dw2t = K.grouped_wgrad(dy3, hid, n_wgroups=W, group_rows=group_rows,
                                   rows_clip=rows_clip, out_dtype=_wgrad_dtype(w23))
            dw1t = K.grouped_wgrad(dz, x3, n_wgroups=W, group_rows=group_rows,
                                   rows_clip=rows_clip, out_dtype=_wgrad_dtype(w13))
            # bias gradients: column sums over the valid rows, both matrices
            # in one launch per pass
            db2_g, db1_g = K.grouped_colsum2(dy3, dz, group_rows, rows_clip)
        db2, db1 = _wsum(db2_g, W), _wsum(db1_g, W)
        return ((dx.view(C, d) if two_d else dx), dw1t.to(w13.dtype).view(w1_shape),
                db1.view(b1_shape), dw2t.to(w23.dtype).view(w2_shape), db2.view(b2_shape),
                (dy if has_res and not fuse_res else None), None, None, None)


class GateFn(torch.autograd.Function):
    """Differentiable part of the gate: returns the kept-selection weights
    (T, k) and aux = N * sum_i f_i P_i (arch.py:436-439, 481-485).  Routing
    (indices, drops, counts) comes in as constants from the gate kernel, and
    so do the probability sums: aux is formed from the kernel's prob_sum, no
    softmax pass.  With noise (arch.py:405-415) the logits carry
    eps * softplus(src W_noise) and the backward differentiates through it
    (noise_pre = src W_noise).  Backward: one kernel (scmoe_gate_backward)."""

    @staticmethod
    def forward(ctx, src, w_gate_t, w_noise_t, logits, indices, counts, weights, prob_sum, k,
                eps, noise_pre):
        t, n = logits.shape
        aux = K.gate_aux_loss(counts, prob_sum, t, k)
        ctx.save_for_backward(src, w_gate_t, w_noise_t, logits, indices, counts, weights, eps,
                              noise_pre)
        return weights.clone(), aux

    @staticmethod
    def backward(ctx, d_weights, d_aux):
        src, w_gate_t, w_noise_t, logits, indices, counts, weights, eps, noise_pre = \
            ctx.saved_tensors
        noise = noise_pre is not None
        need_src = ctx.needs_input_grad[0]
        if d_weights is not None and indices.shape[1] == 1:
            d_weights = None          # top-1: the weight is identically 1 (zero VJP)
        if (d_weights is None and d_aux is None) or logits.shape[1] == 1:
            # one expert: p = f = 1, so the balance loss is constant (zero VJP)
            return (None,) * 11
        d_src, d_wg, d_wn = K.gate_backward(
            src, logits, indices, weights, counts, w_gate_t, d_weights=d_weights, d_aux=d_aux,
            w_noise_t=w_noise_t if noise else None, eps=eps if noise else None,
            noise_pre=noise_pre, need_src=need_src)
        return (d_src if need_src else None, d_wg if ctx.needs_input_grad[1] else None,
                d_wn if (noise and ctx.needs_input_grad[2]) else None) + (None,) * 8


def gate_weights_aux(gate, src: torch.Tensor, dec):
    """(weights, aux) of a routed decision as differentiable functions of the
    source rows and the gate (and noise) weights."""
    noise = gate.noise_enabled and dec.eps is not None
    noise_pre = None
    if noise:
        with torch.no_grad():
            noise_pre = src.float() @ gate.w_noise_t.t()
    return GateFn.apply(src, gate.w_gate_t, gate.w_noise_t if noise else None, dec.logits,
                        dec.indices, dec.counts, dec.weights, dec.prob_sum, dec.k,
                        dec.eps if noise else None, noise_pre)


class DispatchFn(torch.autograd.Function):
    """x_src -> capacity-slotted (E, C, d) buffer with zero-padded tails."""

    @staticmethod
    def forward(ctx, x, indices, slots, kept, n_experts, capacity):
        buf = K.dispatch(x, indices, slots, n_experts, capacity)
        K.zero_tails(buf, kept, capacity)
        ctx.save_for_backward(indices, slots)
        ctx.capacity = capacity
        return buf

    @staticmethod
    def backward(ctx, dbuf):
        indices, slots = ctx.saved_tensors
        ones = torch.ones(indices.shape, device=dbuf.device, dtype=torch.float32)
        dx = K.combine(dbuf.contiguous(), indices, slots, ones, ctx.capacity)
        return dx, None, None, None, None, None


class CombineFn(torch.autograd.Function):
    """out = c_se * se + c_rt * sum_j w_j y[e_j, slot_j] (+ residual) —
    combine (arch.py:380-392) with the routed sum (arch.py:418-433)."""

    @staticmethod
    def forward(ctx, y, se, weights, x_cur, w_cg, residual, indices, slots, kept, capacity, mode,
                link=None):
        out = K.combine(y, indices, slots, weights.contiguous(), capacity, se_out=se, mode=mode,
                        x_cur=x_cur, w_cg=w_cg, residual=residual)
        ctx.save_for_backward(y, se, weights, x_cur, w_cg, indices, slots, kept)
        ctx.meta = (capacity, mode, residual is not None)
        ctx.link = link          # park the residual gradient for the shared FFN's dx GEMM
        return out

    @staticmethod
    def backward(ctx, dout):
        y, se, weights, x_cur, w_cg, indices, slots, kept = ctx.saved_tensors
        capacity, mode, has_res = ctx.meta
        dout = dout.contiguous()
        t, k = indices.shape
        n_exp = y.shape[0]
        d_se = d_xcur = d_wcg = None
        c_rt = None
        if mode == "direct_add":
            d_se = dout if se is not None else None
        else:
            z = x_cur.float() @ w_cg.t()                       # (T, 1|2)
            dse_dot = (dout.float() * se.float()).sum(1)
            if mode == "cg1":
                c = torch.sigmoid(z[:, 0])
                d_se = (c[:, None] * dout.float()).to(dout.dtype)
                dz = (dse_dot * c * (1 - c))[:, None]
            else:
                c = torch.softmax(z, dim=1)
                routed = K.combine(y, indices, slots, weights.contiguous(), capacity)
                drt_dot = (dout.float() * routed.float()).sum(1)
                dc = torch.stack([dse_dot, drt_dot], 1)
                dz = c * (dc - (c * dc).sum(1, keepdim=True))
                d_se = (c[:, :1] * dout.float()).to(dout.dtype)
                c_rt = c[:, 1]
            d_wcg = dz.t() @ x_cur.float()
            d_xcur = (dz @ w_cg).to(x_cur.dtype)
        scale = weights.float() if c_rt is None else weights.float() * c_rt[:, None]
        dy = K.dispatch_scaled(dout, indices, slots, n_exp, capacity, scale)
        K.zero_tails(dy, kept, capacity)
        d_weights = None
        if k > 1:
            # <d routed_t, y[e_j, slot_j]> for kept selections (c_rt folded in)
            gathered = y[indices.long().clamp(max=n_exp - 1), slots.long().clamp(max=capacity - 1)]
            dro = dout.float() if c_rt is None else dout.float() * c_rt[:, None]
            d_weights = (gathered.float() * dro[:, None, :]).sum(-1) * (slots < capacity)
        d_res = dout if has_res else None
        if has_res and ctx.link is not None:
            _park(ctx.link, dout)
            d_res = None
        return (dy, d_se, d_weights, d_xcur, d_wcg, d_res, None, None, None, None, None, None)


class ExchangeFn(torch.autograd.Function):
    """Equal-split all-to-all of a destination-major (E, C, d) buffer; its
    VJP is the reverse all-to-all (ep.exchange_rows is its own transpose)."""

    @staticmethod
    def forward(ctx, buf, group):
        from . import ep
        ctx.group = group
        return ep.exchange_rows(buf, group)

    @staticmethod
    def backward(ctx, d):
        from . import ep
        return ep.exchange_rows(d.contiguous(), ctx.group), None


def _sgd_fusable(p: torch.Tensor) -> bool:
    g = p.grad
    vec = 8 if p.dtype == torch.bfloat16 else 4
    return (p.is_cuda and p.dtype in (torch.bfloat16, torch.float32) and g.dtype == p.dtype
            and p.is_contiguous() and g.is_contiguous() and p.numel() % vec == 0
            and p.data_ptr() % 16 == 0 and g.data_ptr() % 16 == 0)


def sgd_step(params, lr: float) -> None:
    """In-place SGD (the reference's toy trainer, grad.py:330-331): every
    parameter in ONE launch of scmoe_sgd_update (bf16 weights and fp32
    biases alike; torch's multi-tensor apply ran it as ~70 CTAs, 22 us at
    configs[1]).  Parameters the kernel cannot take (odd sizes / alignment)
    go through torch's foreach add, same values."""
    with torch.no_grad():
        fused, rest = [], {}
        for p in params:
            if p.grad is None:
                continue
            if _sgd_fusable(p):
                fused.append(p)
            else:
                rest.setdefault((p.dtype, p.grad.dtype, p.device), []).append(p)
        if fused:
            K.sgd_update(fused, [p.grad for p in fused], lr)
        for ps in rest.values():
            torch._foreach_add_(ps, [p.grad for p in ps], alpha=-lr)


class MeanLossFn(torch.autograd.Function):
    """mean(out) accumulated in fp32 (LossSpec "mean", grad.py:52-67); the
    backward fills the constant gradient in one vectorised pass from the
    device scalar (autograd's MeanBackward expanded it through a
    non-vectorised broadcast kernel plus a dtype cast, ~22 us at configs[1])."""

    @staticmethod
    def forward(ctx, out):
        ctx.shape, ctx.dtype, ctx.n = out.shape, out.dtype, out.numel()
        if out.dtype in (torch.bfloat16, torch.float32) and out.is_contiguous():
            return K.mean_f32(out)
        return out.mean(dtype=torch.float32)

    @staticmethod
    def backward(ctx, g):
        out = torch.empty(ctx.shape, device=g.device, dtype=ctx.dtype)
        if g.dtype == torch.float32 and ctx.dtype in (torch.bfloat16, torch.float32):
            return K.fill_div(out, g.contiguous(), float(ctx.n))   # = (g / n).to(dtype), one pass
        return out.fill_((g / ctx.n).to(ctx.dtype))


def mean_loss(out: torch.Tensor) -> torch.Tensor:
    return MeanLossFn.apply(out)


def allreduce_replicated_grads(module, group=None, experts_sharded: bool = True) -> None:
    """Gradient of the mean of the per-rank objectives, (1/G) sum_r loss_r —
    the objective of training on the ranks' slices together (each rank runs
    the reference's compute_loss on its own slice, grad.py:52-67).

    * Replicated parameters (gate, shared expert, backbone): every rank holds
      d loss_r / dp, so they are all-reduced and divided by G.
    * Sharded routed experts (`experts_sharded`, expert parallelism): the
      owner's weight-gradient GEMM already sums the rows of every source rank
      (the reverse exchange brings each rank's dy to the owner), i.e. it holds
      sum_r d loss_r / dW_e; dividing by G gives the same mean.  Without
      expert parallelism the experts are replicas and are all-reduced like
      everything else."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    ws = dist.get_world_size(group)
    named = [(n, p) for n, p in module.named_parameters() if p.grad is not None]

    def sharded(n):
        return experts_sharded and ".experts." in f".{n}"
    own = [p.grad for n, p in named if sharded(n)]
    if own:
        torch._foreach_div_(own, float(ws))
    grads = [p.grad for n, p in named if not sharded(n)]
    if not grads:
        return
    flat = torch._utils._flatten_dense_tensors(grads)
    dist.all_reduce(flat, group=group)
    flat.div_(ws)
    for g, v in zip(grads, torch._utils._unflatten_dense_tensors(flat, grads)):
        g.copy_(v)
