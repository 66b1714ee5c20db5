"""Host-side behaviour that needs no GPU: config validation, quota rule, and
the product refusing to run on CPU tensors (no fallback)."""

import math

import numpy as np
import pytest
import torch

import paper_2404_05019_b200 as P
from oracle import scmoe_oracle as O


def test_quota_matches_oracle():
    rng = np.random.default_rng(0)
    for _ in range(2000):
        cf = float(rng.uniform(0.05, 4.0))
        t, k, n = int(rng.integers(1, 70000)), int(rng.integers(1, 3)), int(rng.integers(1, 65))
        assert P.expert_quota(cf, t, k, n) == O.expert_quota(cf, t, k, n)


def test_capacity_config_validation():
    with pytest.raises(ValueError):
        P.CapacityConfig(capacity_factor=0)
    with pytest.raises(ValueError):
        P.CapacityConfig(policy="reroute")


def test_layer_config_validation():
    with pytest.raises(P.ConfigError):
        P.ScMoELayer(16, 32, 4, combine_mode="mystery", device="cpu")
    with pytest.raises(P.ConfigError):
        P.ScMoELayer(16, 32, 65, device="cpu")
    with pytest.raises(ValueError):
        P.Top2MoELayer(16, 32, 1, k_routed=2, device="cpu")
    with pytest.raises(P.ConfigError):
        P.ScMoEBlockPair(16, 32, 4, variant="scmoe", shortcut_pos=None, device="cpu")
    with pytest.raises(P.ConfigError):
        P.ScMoEBlockPair(16, 32, 4, variant="standard", combine_mode="cg1", device="cpu")


def test_cpu_tensors_fail_loudly():
    m = P.ScMoELayer(16, 32, 4, dtype=torch.float32, device="cpu")
    x = torch.randn(8, 16)
    with pytest.raises((RuntimeError, ImportError)):
        m(x, x)


def test_from_reference_layout():
    """Weights are stored K-major (transposed) after import."""
    pp = O.init_pair(8, 16, 4, O.Rng(3).spawn(0), variant="scmoe", combine_mode="cg2")
    m = P.ScMoELayer.from_reference(pp.moe, P.CapacityConfig(1.25), dtype=torch.float32,
                                    device="cpu")
    assert m.combine_mode == "cg2" and m.capacity.capacity_factor == 1.25
    np.testing.assert_allclose(m.experts.w1t[2].numpy(), pp.moe.experts[2].w1.T, rtol=1e-6)
    np.testing.assert_allclose(m.shared.w2t.numpy(), pp.moe.shared.w2.T, rtol=1e-6)
    np.testing.assert_allclose(m.gate.w_gate_t.numpy(), pp.moe.gate.w_gate.T, rtol=1e-6)
    np.testing.assert_allclose(m.w_cg.numpy(), pp.moe.w_cg, rtol=1e-6)


def test_peer_exchange_layout_and_tables():
    """p2p EP host logic (no GPU): buffer layout is 256-byte aligned in the
    order recv | y | back | recv_counts | flags, and every peer-table row is
    the peer's base plus that buffer's offset."""
    from paper_2404_05019_b200.ep_p2p import PeerExchange
    world, e_l, cap, d = 4, 2, 100, 64
    sizes, offs, total = PeerExchange.layout(world, e_l, cap, d, torch.bfloat16)
    G = world * e_l
    assert sizes == [G * cap * d * 2] * 3 + [G * 4, 2 * world * 4]
    assert all(o % 256 == 0 for o in offs) and offs == sorted(offs) and total >= offs[-1] + sizes[-1]
    x = PeerExchange(world, 1, e_l, cap, d, torch.bfloat16, "cpu")
    assert x.recv.shape == x.y.shape == x.back.shape == (G, cap, d)
    assert x.flags.numel() == 2 * world and x.epoch.numel() == 4
    bases = [1 << 40, 2 << 40, 3 << 40, 4 << 40]
    x.set_peer_bases(bases)
    for i, o in enumerate(offs):
        assert x.tables[0, i].tolist() == [b + o for b in bases]
    with pytest.raises(ValueError):
        x.set_peer_bases(bases[:2])


def test_peer_exchange_chunked_layout():
    """Chunked pipelining on the p2p backend: `chunks` independent exchanges
    in one storage; chunk c's region i starts c * size_i / chunks after the
    region, back rows are chunk-major (chunks * E, C, d) — the numbering of
    ep.chunk_routing — and the fused-return targets of chunk c point into the
    source's back rows of chunk c."""
    from paper_2404_05019_b200.ep_p2p import PeerExchange
    world, e_l, cc, d, n = 2, 4, 30, 64, 3
    G = world * e_l
    sizes, offs, total = PeerExchange.layout(world, e_l, cc, d, torch.bfloat16, chunks=n)
    assert sizes == [n * G * cc * d * 2] * 3 + [n * G * 4, n * 2 * world * 4]
    x = PeerExchange(world, 1, e_l, cc, d, torch.bfloat16, "cpu", chunks=n)
    assert x.back.shape == (n * G, cc, d) and x.part("back", 2).shape == (G, cc, d)
    assert x.part("recv_counts", 1).numel() == G and x.epoch.numel() == 4 * n
    bases = [1 << 40, 2 << 40]
    x.set_peer_bases(bases)
    for c in range(n):
        for i, o in enumerate(offs):
            assert x.tables[c, i].tolist() == [b + o + c * sizes[i] // n for b in bases]
        row = cc * d * 2
        for g in range(G):
            src, el = divmod(g, e_l)
            assert x.group_out[c, g].item() == (bases[src] + offs[2] + c * sizes[2] // n +
                                                (1 * e_l + el) * row)
    with pytest.raises(ValueError):
        PeerExchange(world, 0, e_l, cc, d, torch.bfloat16, "cpu", chunks=0)


def test_bench_reference_arm_prints_one_json_line():
    """The driver contract: stdout carries exactly one JSON line (fd 1 is
    redirected to stderr for the run, so native banners cannot interleave)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                        "--workload", "swinv2s", "--steps", "1", "--warmup", "0",
                        "--ref-tokens", "16"], capture_output=True, text=True, timeout=600,
                       cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1


def test_bench_model_flops_formula():
    """bench.py model_flops: matmul FLOPs of the configs[2] block pair, by hand.
    Per token: 2 x (QKV 6d^2 + O 2d^2 + causal scores/PV 4 d (S+1)/2) +
    Block-MLP 4dh + shared 4dh + routed 4dh (all kept) + gate 2dN."""
    import importlib.util, os
    spec = importlib.util.spec_from_file_location(
        "bench", os.path.join(os.path.dirname(os.path.dirname(__file__)), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    w = bench.WORKLOADS["gpt3xl"]
    T, d, h, S, N = 16384, 2048, 8192, 2048, 8
    per_tok = 2 * (8 * d * d + 4 * d * (S + 1) / 2) + 3 * 4 * d * h + 2 * d * N
    assert bench.block_pair_flops(w, T, T, N) == pytest.approx(per_tok * T, rel=1e-12)
    # the every-block placement has no Block-MLP and one attention
    wb = bench.WORKLOADS["every_block"]
    d2, h2, S2 = wb["d"], wb["h"], wb["seq"]
    per_tok2 = 8 * d2 * d2 + 4 * d2 * (S2 + 1) / 2 + 2 * 4 * d2 * h2 + 2 * d2 * 16
    assert bench.block_pair_flops(wb, 100, 100, 16) == pytest.approx(per_tok2 * 100, rel=1e-12)
