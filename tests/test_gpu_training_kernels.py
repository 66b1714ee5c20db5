"""K7 backward kernels vs torch fp64 references of the same ops (bf16 inputs,
tolerance 2e-2 scaled by max|ref|): MN-major (transposed-weight) data
gradients, the GELU-backward and pre-activation epilogues, zero-tail padding,
the split-K grouped weight gradient, grouped column sums and the scaled
dispatch used by the combine backward."""

import pytest
import torch

pytestmark = pytest.mark.gpu

K = L = None


def setup_module(module):
    global K, L
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_05019_b200 import _lib, kernels
    K, L = kernels, _lib


def _close(got, ref, rtol=2e-2):
    got, ref = got.double(), ref.double()
    bound = rtol * (ref.abs() + ref.abs().max() + 1e-12)
    err = (got - ref).abs()
    assert (err <= bound).all(), f"max err {err.max().item():.3g}, max ref {ref.abs().max().item():.3g}"


def _gelu_grad(z):
    return 0.5 * (1 + torch.erf(z / 2 ** 0.5)) + z * torch.exp(-0.5 * z * z) / (2 * torch.pi) ** 0.5


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("tile_n", [128, 256])
@pytest.mark.parametrize("G,W,C,Kd,N", [(1, 1, 384, 256, 512), (4, 2, 300, 1536, 384),
                                        (8, 8, 256, 384, 1536)])
def test_dgrad_transposed_weights(mode, tile_n, G, W, C, Kd, N):
    """out = a @ w[g % W]  with w stored (W, k_in, n_out) — MN-major tcgen05 B."""
    K.set_gemm_mode(mode)
    K.set_gemm_tile_n(tile_n)
    try:
        g = torch.Generator(device="cuda").manual_seed(G + N)
        a = torch.randn(G, C, Kd, device="cuda", generator=g).bfloat16()
        w = (torch.randn(W, Kd, N, device="cuda", generator=g) / Kd ** 0.5).bfloat16()
        z = torch.randn(G, C, N, device="cuda", generator=g).bfloat16()
        rows = torch.tensor([max(1, C - 29 * i) for i in range(G)], device="cuda", dtype=torch.int32)
        out = torch.full((G, C, N), float("nan"), device="cuda", dtype=torch.bfloat16)
        K.grouped_gemm_ex(a, w, L.W_KN, N, aux_in=z, epilogue=L.EPI_GELU_BWD, group_rows=rows,
                          rows_clip=C, zero_tail=True, out=out)
        torch.cuda.synchronize()
        for gi in range(G):
            r = int(rows[gi])
            ref = (a[gi, :r].double() @ w[gi % W].double()) * _gelu_grad(z[gi, :r].double())
            _close(out[gi, :r], ref)
            tail_end = min(C, ((r + (255 if mode == 2 else 127)) // (256 if mode == 2 else 128)) * (256 if mode == 2 else 128))
            assert torch.all(out[gi, r:tail_end] == 0)
    finally:
        K.set_gemm_mode(0)
        K.set_gemm_tile_n(0)


def test_forward_preactivation_store():
    g = torch.Generator(device="cuda").manual_seed(7)
    a = torch.randn(2, 200, 256, device="cuda", generator=g).bfloat16()
    w = (torch.randn(2, 512, 256, device="cuda", generator=g) / 16).bfloat16()
    b = torch.randn(2, 512, device="cuda", generator=g)
    zbuf = torch.empty(2, 200, 512, device="cuda", dtype=torch.bfloat16)
    h = K.grouped_gemm_ex(a, w, L.W_NK, 512, bias=b, aux_out=zbuf, epilogue=L.EPI_BIAS_GELU)
    zref = torch.einsum("gck,gnk->gcn", a.double(), w.double()) + b.double()[:, None, :]
    _close(zbuf, zref)
    _close(h, torch.nn.functional.gelu(zref))


@pytest.mark.parametrize("G,W,C,M,N,splits", [(1, 1, 4096, 384, 1536, 0), (8, 8, 700, 1536, 384, 0),
                                              (4, 2, 513, 256, 264, 3), (2, 1, 128, 64, 128, 1),
                                              (16, 2, 300, 384, 1536, 0), (2, 2, 900, 384, 384, 0)])
@pytest.mark.parametrize("mode,tile_n", [(0, 0), (1, 128), (2, 128), (1, 256), (2, 256)])
def test_grouped_wgrad(G, W, C, M, N, splits, mode, tile_n):
    """Split-K weight gradient, every tile shape: auto (least padding of
    (m_out, n_out)), 1-SM 128-row and 2-SM 256-row tiles x BN 128 / 256."""
    K.set_gemm_mode(mode)
    K.set_gemm_tile_n(tile_n)
    try:
        _wgrad_case(G, W, C, M, N, splits)
    finally:
        K.set_gemm_mode(0)
        K.set_gemm_tile_n(0)


def _wgrad_case(G, W, C, M, N, splits):
    g = torch.Generator(device="cuda").manual_seed(G * 3 + M)
    a = torch.randn(G, C, M, device="cuda", generator=g).bfloat16()
    b = torch.randn(G, C, N, device="cuda", generator=g).bfloat16()
    rows = torch.randint(1, C + 1, (G,), device="cuda", generator=g, dtype=torch.int32)
    if G > 1:
        rows[1] = 0
    K.zero_tails(a, rows, C)
    K.zero_tails(b, rows, C)
    out = K.grouped_wgrad(a, b, n_wgroups=W, group_rows=rows, rows_clip=C, splits=splits)
    torch.cuda.synchronize()
    rr = rows.tolist()
    for w in range(W):
        ref = torch.zeros(M, N, dtype=torch.float64, device="cuda")
        for gi in range(w, G, W):
            r = rr[gi]
            ref += a[gi, :r].double().t() @ b[gi, :r].double()
        _close(out[w] if out.dim() == 3 else out, ref, rtol=1e-2)


@pytest.mark.parametrize("splits", [0, 1, 3])
def test_grouped_wgrad_bf16_out(splits):
    """bf16 output = the fp32 result rounded once (same bits as .to(bf16))."""
    g = torch.Generator(device="cuda").manual_seed(9 + splits)
    a = torch.randn(4, 640, 384, device="cuda", generator=g).bfloat16()
    b = torch.randn(4, 640, 1536, device="cuda", generator=g).bfloat16()
    f32 = K.grouped_wgrad(a, b, n_wgroups=2, splits=splits)
    b16 = K.grouped_wgrad(a, b, n_wgroups=2, splits=splits, out_dtype=torch.bfloat16)
    assert b16.dtype == torch.bfloat16
    assert torch.equal(b16, f32.to(torch.bfloat16))


def test_zero_tails_and_colsum():
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(3, 300, 128, device="cuda", generator=g).bfloat16()
    rows = torch.tensor([10, 64, 250], device="cuda", dtype=torch.int32)
    K.zero_tails(x, rows, 300, align=64)
    assert torch.all(x[0, 10:64] == 0) and torch.all(x[2, 250:256] == 0)
    assert not torch.all(x[0, 64:70] == 0)          # beyond the padding: untouched
    s = K.grouped_colsum(x, rows, 300)
    for gi, r in enumerate(rows.tolist()):
        torch.testing.assert_close(s[gi], x[gi, :r].float().sum(0), rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("G,C,D0,D1", [(1, 18432, 384, 1536), (3, 300, 128, 2048), (8, 77, 8, 16)])
def test_colsum2_matches_two_colsums(dtype, G, C, D0, D1):
    """Both bias gradients of an FFN in one launch per pass: the same values
    as two single-matrix calls (same stripes per matrix only when the tile
    counts agree, so compared at fp32 tolerance) and torch sums."""
    g = torch.Generator(device="cuda").manual_seed(G + D1)
    a = torch.randn(G, C, D0, device="cuda", generator=g).to(dtype)
    b = torch.randn(G, C, D1, device="cuda", generator=g).to(dtype)
    rows = torch.randint(0, C + 1, (G,), device="cuda", generator=g, dtype=torch.int32)
    s0, s1 = K.grouped_colsum2(a, b, rows, C)
    for gi, r in enumerate(rows.tolist()):
        torch.testing.assert_close(s0[gi], a[gi, :r].double().sum(0).float(), rtol=1e-4, atol=2e-3)
        torch.testing.assert_close(s1[gi], b[gi, :r].double().sum(0).float(), rtol=1e-4, atol=2e-3)
    torch.testing.assert_close(s0, K.grouped_colsum(a, rows, C), rtol=1e-5, atol=1e-3)


def test_dispatch_scaled():
    g = torch.Generator(device="cuda").manual_seed(2)
    T, d, N, k = 500, 256, 4, 2
    x = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    w = torch.randn(N, d, device="cuda", generator=g)
    quota = K.expert_quota(1.0, T, k, N)
    dec = K.gate_topk(x, w, k, quota)
    scale = torch.rand(T, k, device="cuda", generator=g)
    buf = torch.zeros(N, quota, d, device="cuda", dtype=torch.bfloat16)
    K.dispatch_scaled(x, dec.indices, dec.slots, N, quota, scale, out=buf)
    idx, sl = dec.indices.long(), dec.slots.long()
    kept = sl < quota
    tt = torch.arange(T, device="cuda")[:, None].expand(T, k)
    ref = torch.zeros(N, quota, d, device="cuda", dtype=torch.float64)
    ref[idx[kept], sl[kept]] = x[tt[kept]].double() * scale[kept].double()[:, None]
    _close(buf, ref, rtol=1e-2)


@pytest.mark.parametrize("G,W,C,N", [(1, 1, 18432, 384), (8, 8, 700, 1536), (4, 2, 300, 264)])
def test_bias_grad_tensor_core(G, W, C, N):
    g = torch.Generator(device="cuda").manual_seed(C)
    dy = torch.randn(G, C, N, device="cuda", generator=g).bfloat16()
    rows = torch.randint(1, C + 1, (G,), device="cuda", generator=g, dtype=torch.int32)
    K.zero_tails(dy, rows, C)
    out = K.bias_grad(dy, n_wgroups=W, group_rows=rows, rows_clip=C)
    for w in range(W):
        ref = sum(dy[gi, :int(rows[gi])].double().sum(0) for gi in range(w, G, W))
        _close(out[w], ref, rtol=1e-3)


def test_sgd_update_matches_foreach():
    """scmoe_sgd_update (one launch over every parameter) gives the values of
    torch._foreach_add_(p, g, alpha=-lr): fp32 arithmetic, rounded once."""
    from paper_2404_05019_b200 import training as TR
    g = torch.Generator(device="cuda").manual_seed(3)
    shapes = [((384, 1536), torch.bfloat16), ((1536,), torch.float32), ((8, 384), torch.float32),
              ((3, 384, 384), torch.bfloat16), ((7,), torch.bfloat16)]     # 7: torch path
    ps = [torch.randn(s, device="cuda", generator=g).to(dt) for s, dt in shapes]
    gs = [torch.randn(s, device="cuda", generator=g).to(dt) for s, dt in shapes]
    ref = [p.clone() for p in ps]
    torch._foreach_add_(ref, gs, alpha=-0.03)
    params = [torch.nn.Parameter(p) for p in ps]
    for p, gr in zip(params, gs):
        p.grad = gr
    TR.sgd_step(params, 0.03)
    for p, r in zip(params, ref):
        assert torch.equal(p.data, r)


def test_mean_loss_gradient():
    from paper_2404_05019_b200 import training as TR
    x = torch.randn(300, 64, device="cuda").bfloat16().requires_grad_(True)
    l = TR.mean_loss(x)
    l.backward()
    x2 = x.detach().clone().requires_grad_(True)
    l2 = x2.mean(dtype=torch.float32)
    l2.backward()
    # the loss is our deterministic two-pass fp32 mean (another summation
    # order than torch's); the gradient fill is bit-identical
    torch.testing.assert_close(l, l2, rtol=1e-5, atol=1e-7)
    assert torch.equal(x.grad, x2.grad)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("n", [1, 7, 8, 1000, 18432 * 384 + 3])
def test_fill_div_matches_torch(dtype, n):
    """The mean-loss backward's constant gradient: bit-identical to
    (g / n).to(dtype) broadcast by torch."""
    g = torch.tensor(0.7310585, device="cuda", dtype=torch.float32)
    out = torch.empty(n, device="cuda", dtype=dtype)
    K.fill_div(out, g, float(n))
    ref = torch.empty(n, device="cuda", dtype=dtype).fill_((g / n).to(dtype))
    assert torch.equal(out, ref)


def test_gate_aux_loss_matches_formula():
    g = torch.Generator(device="cuda").manual_seed(4)
    counts = torch.randint(0, 500, (8,), device="cuda", generator=g, dtype=torch.int32)
    ps = torch.rand(8, device="cuda", generator=g) * 100
    T, k = 1000, 2
    aux = K.gate_aux_loss(counts, ps, T, k)
    ref = 8 * ((counts.double() / (T * k)) * (ps.double() / T)).sum()
    torch.testing.assert_close(aux.double(), ref, rtol=1e-6, atol=0)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("n", [1, 5, 300, 18432 * 384, 1000003])
def test_mean_f32(dtype, n):
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randn(n, device="cuda", generator=g).to(dtype)
    m = K.mean_f32(x)
    torch.testing.assert_close(m.double(), x.double().mean(), rtol=1e-5, atol=1e-6)
    assert torch.equal(m, K.mean_f32(x))          # deterministic
    off = K.mean_f32(x[1:]) if n > 1 else None   # unaligned start: the scalar path
    if off is not None:
        torch.testing.assert_close(off.double(), x[1:].double().mean(), rtol=1e-5, atol=1e-6)


def test_gate_sync_words_left_zero():
    """scmoe_gate_topk_ex with caller-kept sync words: identical decisions to
    the per-call memset path, words zero after every launch."""
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(5000, 256, device="cuda", generator=g).bfloat16()
    w = torch.randn(8, 256, device="cuda", generator=g) / 16
    quota = K.expert_quota(1.0, 5000, 2, 8)
    sync = torch.zeros(4, device="cuda", dtype=torch.int32)
    a = K.gate_topk(x, w, 2, quota)
    for _ in range(3):
        b = K.gate_topk(x, w, 2, quota, sync=sync)
        assert torch.equal(a.slots, b.slots) and torch.equal(a.indices, b.indices)
        assert torch.equal(a.counts, b.counts) and torch.equal(a.prob_sum, b.prob_sum)
        assert int(sync.abs().sum()) == 0
