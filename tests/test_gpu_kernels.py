"""Kernel-level parity on the B200, through the C ABI.

Gate: bit-exact expert index, capacity slot and drop flag against the
oracle's select_topk + apply_capacity (gating.py:110-156) run on the
kernel's own fp32 logits upcast to float64 (ties -> lowest index, signed
zeros, T not a multiple of the tile).  GEMM / dispatch / combine: against
torch fp32/fp64 references of the same op (tolerances stated per test).
"""

import numpy as np
import pytest
import torch

from oracle import scmoe_oracle as O

pytestmark = pytest.mark.gpu

K = None


def setup_module(module):
    global K
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_05019_b200 import kernels
    K = kernels


def _gate_case(T, d, N, k, cf, dtype, seed, ties=False, zeros=False, noise=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(T, d, device="cuda", generator=g).to(dtype)
    w = torch.randn(N, d, device="cuda", generator=g) / d ** 0.5
    if ties and N >= 3:
        w[N - 1] = w[0]          # identical columns -> bit-identical logits
        w[1] = w[N - 2]
    if zeros:
        x[::3] = 0               # all-zero logits rows: every expert ties
    wn = eps = None
    if noise:
        wn = torch.randn(N, d, device="cuda", generator=g) / d ** 0.5
        eps = torch.randn(T, N, device="cuda", generator=g)
    quota = K.expert_quota(cf, T, k, N)
    out = K.gate_topk(x, w, k, quota, w_noise_t=wn, eps=eps)
    torch.cuda.synchronize()
    h = out.logits.double().cpu().numpy()
    ref = O.apply_capacity(O.select_topk(h, k), cf, N, T)
    np.testing.assert_array_equal(out.indices.long().cpu().numpy(), ref.indices)
    np.testing.assert_array_equal(out.dropped.bool().cpu().numpy(), ref.dropped)
    slots = O.capacity_slots(ref.indices, N)
    np.testing.assert_array_equal(out.slots.long().cpu().numpy(), slots)
    np.testing.assert_allclose(out.weights.double().cpu().numpy(), ref.weights, rtol=2e-6, atol=1e-7)
    np.testing.assert_array_equal(out.counts.long().cpu().numpy(),
                                  np.bincount(ref.indices.ravel(), minlength=N))
    p = O.row_softmax(h).sum(axis=0)
    np.testing.assert_allclose(out.prob_sum.double().cpu().numpy(), p, rtol=1e-4, atol=1e-3)
    # logits vs a plain fp32 torch reference of the same op
    hl = x.float() @ w.t()
    if noise:
        hl = hl + eps * torch.nn.functional.softplus(x.float() @ wn.t())
    torch.testing.assert_close(out.logits, hl, rtol=1e-4, atol=1e-4)
    return out


@pytest.mark.parametrize("T,d,N,k,cf", [
    (1, 8, 1, 1, 1.0), (7, 16, 3, 2, 0.5), (64, 32, 8, 1, 1.0), (65, 64, 8, 2, 1.0),
    (1000, 256, 8, 1, 1.0), (4097, 128, 16, 2, 1.25), (16384, 2048, 8, 1, 2.0),
    (16384, 2048, 8, 2, 2.0), (3000, 64, 33, 4, 0.75), (2048, 96, 64, 8, 0.3),
    (512, 256, 8, 1, 0.25)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_gate_bit_exact(T, d, N, k, cf, dtype):
    _gate_case(T, d, N, k, cf, dtype, seed=T * 31 + N)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_gate_ties_and_zeros(dtype):
    out = _gate_case(777, 64, 6, 2, 1.0, dtype, seed=5, ties=True, zeros=True)
    idx = out.indices.long().cpu().numpy()
    assert (idx[::3, 0] == 0).all() and (idx[::3, 1] == 1).all()   # all-tied rows


@pytest.mark.parametrize("T,d,N,k,cf", [
    (1, 64, 1, 1, 1.0), (300, 384, 8, 1, 1.0), (129, 320, 5, 2, 1.0), (2000, 4096, 16, 2, 1.0),
    (5000, 3072, 12, 1, 1.25), (64, 64, 16, 4, 0.5), (40000, 256, 8, 2, 1.0),
    (300, 200, 8, 1, 1.0), (129, 72, 5, 2, 1.0), (200000, 64, 8, 2, 1.0)])
def test_gate_tensor_core_path(T, d, N, k, cf):
    """bf16 tokens, N <= 16, d % 64 == 0: the persistent tensor-core gate
    (mma.sync on a 3-part bf16 weight split, bulk-copied row stages): one and
    several stages per tile, partial last stage (d=384, 320), partial last
    tile, more tiles than SMs (T=40000), more CTA-local ranks than the
    shared-memory rank cache holds (T=200000, k=2: re-read from `slots`).
    d % 64 != 0 takes the FMA kernel."""
    _gate_case(T, d, N, k, cf, torch.bfloat16, seed=T + d + N)


def test_gate_tensor_core_matches_fma_path():
    """Same decisions from both logit kernels wherever their fp32 logits agree;
    logits within a few fp32 ulps of each other."""
    import ctypes
    from paper_2404_05019_b200 import _lib
    flag = ctypes.c_int.in_dll(_lib.lib(), "scmoe_gate_force_fma")
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(16384, 2048, device="cuda", generator=g).bfloat16()
    w = torch.randn(8, 2048, device="cuda", generator=g) / 2048 ** 0.5
    quota = K.expert_quota(2.0, 16384, 1, 8)
    try:
        flag.value = 1
        a = K.gate_topk(x, w, 1, quota)
        flag.value = 0
        b = K.gate_topk(x, w, 1, quota)
    finally:
        flag.value = 0
    torch.cuda.synchronize()
    torch.testing.assert_close(a.logits, b.logits, rtol=1e-4, atol=1e-4)
    same = (a.indices == b.indices).float().mean().item()
    assert same > 0.999


def test_gate_noise():
    _gate_case(1500, 128, 8, 2, 1.0, torch.float32, seed=9, noise=True)


def test_gate_rejects_bad_args():
    x = torch.randn(8, 16, device="cuda")
    w = torch.randn(4, 16, device="cuda")
    with pytest.raises(ValueError):
        K.gate_topk(x, w, 5, 4)
    with pytest.raises(ValueError):
        K.gate_topk(torch.randn(8, 10, device="cuda"), torch.randn(4, 10, device="cuda"), 1, 4)


def _ref_ffn_rows(a, wt, bias, gelu):
    y = a.double() @ wt.double().t()
    if bias is not None:
        y = y + bias.double()
    if gelu:
        y = torch.nn.functional.gelu(y)
    return y


@pytest.mark.parametrize("G,W,C,Kd,N", [
    (1, 1, 128, 64, 256), (1, 1, 300, 200, 136), (8, 8, 512, 256, 1024), (4, 2, 130, 72, 520),
    (8, 8, 1024, 2048, 8192), (3, 3, 257, 1024, 264), (16, 16, 64, 384, 1536),
    (1, 1, 256, 128, 128), (1, 1, 256, 128, 384), (1, 1, 1000, 384, 1152),
    (2, 2, 300, 128, 200), (1, 1, 256, 64, 32)])
@pytest.mark.parametrize("gelu", [False, True])
@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("tile_n", [128, 192, 256])
def test_grouped_gemm_bf16(G, W, C, Kd, N, gelu, mode, tile_n):
    """Both tcgen05 variants (1-SM 128xBN, 2-SM cta_group::2 256xBN) at every
    tile width (BN = 256; 192, the exact cover of n_out = 384 / 1152; 128
    with four accumulator stages), with and without the residual epilogue
    (bias + residual runs the straight-line residual path)."""
    K.set_gemm_mode(mode)
    K.set_gemm_tile_n(tile_n)
    try:
        _grouped_gemm_case(G, W, C, Kd, N, gelu,
                           residual=(mode == 2 and gelu) or (not gelu and tile_n != 128))
    finally:
        K.set_gemm_mode(0)
        K.set_gemm_tile_n(0)


def _grouped_gemm_case(G, W, C, Kd, N, gelu, residual):
    g = torch.Generator(device="cuda").manual_seed(G * 7 + C)
    a = torch.randn(G, C, Kd, device="cuda", generator=g).bfloat16()
    wt = (torch.randn(W, N, Kd, device="cuda", generator=g) / Kd ** 0.5).bfloat16()
    bias = torch.randn(W, N, device="cuda", generator=g) * 0.1
    rows = torch.randint(0, C + 40, (G,), device="cuda", generator=g, dtype=torch.int32)
    rows[0] = C + 7   # clipped to C
    if G > 1:
        rows[1] = 0   # empty group
    out = torch.full((G, C, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    res = torch.randn(G, C, N, device="cuda", generator=g).bfloat16() if residual else None
    K.grouped_gemm(a, wt, bias, group_rows=rows, rows_clip=C, gelu=gelu, out=out, residual=res)
    torch.cuda.synchronize()
    rr = rows.clamp(max=C).cpu().tolist()
    for gi in range(G):
        r = rr[gi]
        if r == 0:
            assert torch.isnan(out[gi].float()).all()
            continue
        ref = _ref_ffn_rows(a[gi, :r], wt[gi % W], bias[gi % W], gelu)
        if res is not None:
            ref = ref + res[gi, :r].double()
        got = out[gi, :r].double()
        # bf16 output: |err| <= 2e-2 * (|ref| + max|ref|)
        tol = 2e-2 * (ref.abs() + ref.abs().max())
        assert ((got - ref).abs() <= tol).all(), (gi, (got - ref).abs().max().item())
        if r < C:
            assert torch.isnan(out[gi, r:].float()).all()   # rows past the count untouched


@pytest.mark.parametrize("G,C,Kd,N", [(1, 100, 60, 70), (4, 129, 256, 1024), (8, 64, 256, 1024)])
def test_grouped_gemm_f32(G, C, Kd, N):
    g = torch.Generator(device="cuda").manual_seed(C)
    a = torch.randn(G, C, Kd, device="cuda", generator=g)
    wt = torch.randn(G, N, Kd, device="cuda", generator=g) / Kd ** 0.5
    bias = torch.randn(G, N, device="cuda", generator=g)
    rows = torch.tensor([C - 3 * i for i in range(G)], device="cuda", dtype=torch.int32)
    res = torch.randn(G, C, N, device="cuda", generator=g)
    out = K.grouped_gemm(a, wt, bias, group_rows=rows, rows_clip=C, gelu=True, residual=res)
    for gi in range(G):
        r = C - 3 * gi
        ref = _ref_ffn_rows(a[gi, :r], wt[gi], bias[gi], True) + res[gi, :r].double()
        torch.testing.assert_close(out[gi, :r].double(), ref, rtol=1e-5, atol=1e-5)


def test_dense_gemm_matches_torch_large():
    """Dense (single-group, no row counts) path used by the shared expert."""
    g = torch.Generator(device="cuda").manual_seed(1)
    T, d, h = 4096, 2048, 8192
    x = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    w1t = (torch.randn(h, d, device="cuda", generator=g) / d ** 0.5).bfloat16()
    b1 = torch.zeros(h, device="cuda")
    w2t = (torch.randn(d, h, device="cuda", generator=g) / d ** 0.5).bfloat16()
    b2 = torch.randn(d, device="cuda", generator=g)
    y = K.expert_ffn(x, w1t, b1, w2t, b2)
    hid = torch.nn.functional.gelu(x.float() @ w1t.float().t()).bfloat16()
    ref = hid.float() @ w2t.float().t() + b2
    err = (y.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item(), err


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("k", [1, 2])
def test_dispatch_and_combine(dtype, k):
    g = torch.Generator(device="cuda").manual_seed(k)
    T, d, N = 999, 256, 8
    x = torch.randn(T, d, device="cuda", generator=g).to(dtype)
    w = torch.randn(N, d, device="cuda", generator=g) / d ** 0.5
    quota = K.expert_quota(0.75, T, k, N)
    dec = K.gate_topk(x, w, k, quota)
    buf = torch.zeros(N, quota, d, device="cuda", dtype=dtype)
    K.dispatch(x, dec.indices, dec.slots, N, quota, out=buf)
    idx, sl = dec.indices.long(), dec.slots.long()
    kept = sl < quota
    ref_buf = torch.zeros_like(buf)
    tt = torch.arange(T, device="cuda")[:, None].expand(T, k)
    ref_buf[idx[kept], sl[kept]] = x[tt[kept]]
    assert torch.equal(buf, ref_buf)
    # combine in every mode, with / without residual
    y = torch.randn(N, quota, d, device="cuda", generator=g).to(dtype)
    se = torch.randn(T, d, device="cuda", generator=g).to(dtype)
    res = torch.randn(T, d, device="cuda", generator=g).to(dtype)
    routed = torch.zeros(T, d, device="cuda", dtype=torch.float64)
    for j in range(k):
        m = kept[:, j]
        routed[m] += dec.weights[m, j, None].double() * y[idx[m, j], sl[m, j]].double()
    for mode, rows in (("direct_add", 0), ("cg1", 1), ("cg2", 2)):
        wcg = torch.randn(max(rows, 1), d, device="cuda", generator=g) / d ** 0.5
        z = x.double() @ wcg.double().t()
        if mode == "direct_add":
            ref = se.double() + routed
        elif mode == "cg1":
            ref = torch.sigmoid(z[:, :1]) * se.double() + routed
        else:
            c = torch.softmax(z, dim=1)
            ref = c[:, :1] * se.double() + c[:, 1:2] * routed
        for r in (None, res):
            out = K.combine(y, dec.indices, dec.slots, dec.weights, quota, se_out=se, mode=mode,
                            x_cur=x, w_cg=wcg if rows else None, residual=r)
            expect = ref + (r.double() if r is not None else 0)
            tol = 1e-5 if dtype == torch.float32 else 2e-2
            torch.testing.assert_close(out.double(), expect, rtol=tol, atol=tol * expect.abs().max().item())
    # moe_standard: no shared expert
    out = K.combine(y, dec.indices, dec.slots, dec.weights, quota)
    tol = 1e-5 if dtype == torch.float32 else 2e-2
    torch.testing.assert_close(out.double(), routed, rtol=tol, atol=tol * routed.abs().max().item())


def test_pack_heads_matches_torch():
    """scmoe_pack_heads: strided (B, H, S, hd) sources -> (B, S, n, H, hd)."""
    B, H, S, hd = 3, 5, 70, 32
    base = torch.randn(B, S, 3, H, hd, device="cuda").bfloat16()
    srcs = [base[:, :, i].transpose(1, 2) for i in range(3)]          # BSHD strides
    srcs[1] = srcs[1].contiguous()                                     # BHSD contiguous
    out = K.pack_heads(srcs)
    ref = torch.stack([t.transpose(1, 2) for t in srcs], dim=2)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    one = K.pack_heads([srcs[1]])
    assert torch.equal(one[:, :, 0], srcs[1].transpose(1, 2))


def test_gate_presplit_equals_per_call_split():
    """scmoe_gate_topk_presplit with a cached weight split gives the same
    decision as the per-call split; Top1Gate re-splits after an in-place
    weight update (weight version changes)."""
    import paper_2404_05019_b200 as P
    T, d, N = 3000, 512, 8
    x = torch.randn(T, d, device="cuda").bfloat16()
    w = torch.randn(N, d, device="cuda") / d ** 0.5
    quota = K.expert_quota(1.0, T, 1, N)
    a = K.gate_topk(x, w, 1, quota)
    b = K.gate_topk(x, w, 1, quota, w_split=K.gate_split_weights(w))
    torch.cuda.synchronize()
    for f in ("logits", "indices", "slots", "dropped", "counts", "weights"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f
    gate = P.Top1Gate(d, N, capacity_factor=1.0)
    with torch.no_grad():
        d1 = gate(x)
        s1 = gate._split
        gate.w_gate_t.mul_(-1.0)                 # in-place update: new version
        d2 = gate(x)
    assert gate._split is not s1
    ref = K.gate_topk(x, gate.w_gate_t, 1, quota)
    torch.cuda.synchronize()
    assert torch.equal(d2.indices, ref.indices) and torch.equal(d2.slots, ref.slots)
    assert not torch.equal(d1.indices, d2.indices)


@pytest.mark.parametrize("T,d,N,k", [(65536, 2048, 16, 2), (3000, 4096, 12, 1)])
def test_gate_tensor_core_sync_words_wide(T, d, N, k):
    """The streamed-blob tensor-core gate (N > 8) with caller-kept sync words,
    called repeatedly: the same decisions as the per-call-memset path, the
    words left zero."""
    g = torch.Generator(device="cuda").manual_seed(T + N)
    x = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    w = torch.randn(N, d, device="cuda", generator=g) / d ** 0.5
    quota = K.expert_quota(1.0, T, k, N)
    ref = K.gate_topk(x, w, k, quota)
    sync = torch.zeros(2, device="cuda", dtype=torch.int32)
    for _ in range(3):
        out = K.gate_topk(x, w, k, quota, sync=sync)
        assert torch.equal(out.slots, ref.slots) and torch.equal(out.indices, ref.indices)
        assert torch.equal(out.dropped, ref.dropped) and torch.equal(out.counts, ref.counts)
        assert int(sync.abs().sum()) == 0
