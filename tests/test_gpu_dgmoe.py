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
