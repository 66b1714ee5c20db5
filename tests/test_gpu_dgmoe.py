"""DGMoE (dual top-1 gating, arch.py:447-460, 507-533) on the GPU vs the
float64 oracle (pinned to the reference's DGMoE outputs): routing bit-exact
on the kernels' logits, outputs with routing pinned (fp32 rtol 1e-4, bf16
2e-2, scaled by max|ref|)."""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import scmoe_oracle as O

pytestmark = pytest.mark.gpu
P = None


def setup_module(module):
    global P
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2404_05019_b200 as pkg
    P = pkg


def _t(a, dtype):
    return torch.as_tensor(np.asarray(a), device="cuda").to(dtype).contiguous()


def _pin(dec):
    return dec.indices.long().cpu().numpy(), dec.dropped.cpu().numpy()


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("constraint", [True, False])
@pytest.mark.parametrize("cf", [1.0, 0.5])
def test_dgmoe_layer(dtype, constraint, cf):
    T, d, h, N = 384, 128, 256, 6
    pp = O.init_pair(d, h, N, O.Rng(31).spawn(0), variant="dgmoe")
    x_cur = O.Rng(31).spawn(1).normal((T, d))
    x_prev = x_cur + 0.3 * O.Rng(31).spawn(2).normal((T, d))     # correlated: many clashes
    layer = P.DGMoELayer.from_reference(pp.moe, P.CapacityConfig(cf), constraint=constraint,
                                        dtype=dtype)
    xc, xp = _t(x_cur, dtype), _t(x_prev, dtype)
    out, dc, dp, aux = layer(xc, xp)
    torch.cuda.synchronize()
    # routing bit-exact against dual_routing on the kernels' own logits
    rc, rp = O.dual_routing(dc.logits.double().cpu().numpy(), dp.logits.double().cpu().numpy(),
                            constraint, cf)
    np.testing.assert_array_equal(dc.indices.long().cpu().numpy(), rc.indices)
    np.testing.assert_array_equal(dc.dropped.cpu().numpy(), rc.dropped)
    np.testing.assert_array_equal(dp.indices.long().cpu().numpy(), rp.indices)
    np.testing.assert_array_equal(dp.dropped.cpu().numpy(), rp.dropped)
    if constraint:
        assert (dc.indices[:, 0] != dp.indices[:, 0]).all()
    ref, _, _, raux = O.moe_dual_gating(xc.double().cpu().numpy(), xp.double().cpu().numpy(),
                                        pp.moe, cf, constraint, pinned=(_pin(dc), _pin(dp)))
    rtol = 1e-4 if dtype == torch.float32 else 2e-2
    ok, worst = O.allclose_scaled(out.double().cpu().numpy(), ref, rtol)
    assert ok, worst
    assert float(aux) == pytest.approx(raux, rel=rtol, abs=1e-4)


def test_dgmoe_block_pair_fp32():
    T, d, h, N, cf = 256, 128, 256, 4, 1.0
    pp = O.init_pair(d, h, N, O.Rng(33).spawn(0), variant="dgmoe")
    cfg = SimpleNamespace(d_model=d, d_hidden=h, n_experts=N, variant="dgmoe", shortcut_pos="pos2",
                          k_routed=1, combine_mode="direct_add", capacity_factor=cf,
                          noise_enabled=False, pre_layernorm=False, dgmoe_constraint=True)
    blk = P.ScMoEBlockPair.from_reference(cfg, SimpleNamespace(attn=pp.attn_prev, feed=pp.mlp_prev),
                                          SimpleNamespace(attn=pp.attn_cur, feed=pp.moe),
                                          dtype=torch.float32)
    tokens = O.Rng(33).spawn(1).normal((T, d))
    out, (dc, dp), aux = blk(_t(tokens, torch.float32))
    ref, _, _, raux = O.dgmoe_pair_forward(pp, tokens, cf, True, pinned=(_pin(dc), _pin(dp)))
    ok, worst = O.allclose_scaled(out.double().cpu().numpy(), ref, 1e-4)
    assert ok, worst
    assert float(aux) == pytest.approx(raux, rel=1e-4, abs=1e-5)


def test_dgmoe_trains():
    blk = P.ScMoEBlockPair(128, 256, 4, variant="dgmoe", n_heads=2, seq_len=128,
                           capacity_factor=1.0, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(8))
    blk.requires_grad_(True)
    x = torch.randn(256, 128, device="cuda").bfloat16()
    tgt = torch.randn(256, 128, device="cuda").bfloat16()
    losses = [float(blk.train_step(x, lr=2e-3, target=tgt)) for _ in range(6)]
    assert np.all(np.isfinite(losses)) and losses[-1] < losses[0]
    assert blk.moe.experts.w1t.grad is not None


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_dgmoe_noise_and_replay(dtype):
    """Dual gating with the noisy gate: the two gatings' draws (eps, eps_prev)
    enter the logits (arch.py:514-515); routing is bit-exact on the kernels'
    logits, the output matches the oracle with the same draws, and a replay
    of (eps, eps_prev, indices, dropped, indices_prev, dropped_prev) through
    MoEReplay reproduces the output bit for bit (arch.py:518-520)."""
    T, d, h, N, cf = 384, 128, 256, 6, 1.0
    pp = O.init_pair(d, h, N, O.Rng(37).spawn(0), variant="dgmoe", noise_enabled=True)
    x_cur = O.Rng(37).spawn(1).normal((T, d))
    x_prev = x_cur + 0.3 * O.Rng(37).spawn(2).normal((T, d))
    eps = O.Rng(37).spawn(3).normal((T, N))
    eps_prev = O.Rng(37).spawn(4).normal((T, N))
    layer = P.DGMoELayer.from_reference(pp.moe, P.CapacityConfig(cf), dtype=dtype)
    assert layer.noise_enabled
    xc, xp = _t(x_cur, dtype), _t(x_prev, dtype)
    out, dc, dp, aux = layer(xc, xp, eps=_t(eps, torch.float32), eps_prev=_t(eps_prev, torch.float32))
    torch.cuda.synchronize()
    rc, rp = O.dual_routing(dc.logits.double().cpu().numpy(), dp.logits.double().cpu().numpy(),
                            True, cf)
    np.testing.assert_array_equal(dc.indices.long().cpu().numpy(), rc.indices)
    np.testing.assert_array_equal(dp.indices.long().cpu().numpy(), rp.indices)
    np.testing.assert_array_equal(dc.dropped.cpu().numpy(), rc.dropped)
    ref, _, _, raux = O.moe_dual_gating(xc.double().cpu().numpy(), xp.double().cpu().numpy(),
                                        pp.moe, cf, True, pinned=(_pin(dc), _pin(dp)),
                                        eps=eps, eps_prev=eps_prev)
    rtol = 1e-4 if dtype == torch.float32 else 2e-2
    ok, worst = O.allclose_scaled(out.double().cpu().numpy(), ref, rtol)
    assert ok, worst
    # the noise changes routing vs the clean gate
    clean = O.dual_routing(*(O.gate_logits(z, O.Gate(pp.moe.gate.w_gate, pp.moe.gate.w_noise,
                                                     1, False))[0]
                             for z in (xc.double().cpu().numpy(), xp.double().cpu().numpy())),
                           True, cf)[0]
    assert (clean.indices != rc.indices).any()
    # replay: pinned routing and draws through MoEReplay
    r = P.MoEReplay(eps=eps, indices=dc.indices.long().cpu().numpy(),
                    dropped=dc.dropped.cpu().numpy(), eps_prev=eps_prev,
                    indices_prev=dp.indices.long().cpu().numpy(),
                    dropped_prev=dp.dropped.cpu().numpy())
    out2, dc2, dp2, _ = layer(xc, xp, replay=r)
    assert torch.equal(dc2.indices, dc.indices) and torch.equal(dp2.indices, dp.indices)
    assert torch.equal(out2, out)


def test_dgmoe_block_noise_draws():
    """A noisy DGMoE block pair draws its own noise when none is given (the
    C API needs w_noise and eps together) and trains."""
    blk = P.ScMoEBlockPair(128, 256, 4, variant="dgmoe", n_heads=2, seq_len=128,
                           capacity_factor=1.0, noise_enabled=True, dtype=torch.bfloat16,
                           generator=torch.Generator(device="cuda").manual_seed(9))
    x = torch.randn(256, 128, device="cuda").bfloat16()
    with torch.no_grad():
        out, (dc, dp), aux = blk(x)
    assert dc.eps is not None and dp.eps is not None
    assert torch.isfinite(out.float()).all()
    blk.requires_grad_(True)
    loss = blk.train_step(x, lr=1e-3)
    assert torch.isfinite(loss).item()
    assert blk.moe.gate.w_noise_t.grad is not None
