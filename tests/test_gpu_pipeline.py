"""Chunked pipelining (standard_pipeline / scmoe_overlap_pipeline,
distsim.py:277-300, 358-364): splitting dispatch / expert / combine into
chunks changes the schedule, never the result — chunked forwards equal the
unchunked ones bit for bit (GEMM rows are independent)."""

import pytest
import torch

pytestmark = pytest.mark.gpu
P = None


def setup_module(module):
    global P
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2404_05019_b200 as pkg
    P = pkg


@pytest.mark.parametrize("variant,k,cf", [("scmoe", 1, 2.0), ("standard", 2, 1.0),
                                          ("scmoe", 1, 0.6), ("shared", 2, 1.25)])
@pytest.mark.parametrize("chunks", [2, 3, 4])
def test_chunked_equals_unchunked(variant, k, cf, chunks):
    T, d, h, N = 1024, 256, 512, 8
    kw = dict(variant=variant, k_routed=k, shortcut_pos="pos2" if variant == "scmoe" else None,
              n_heads=4, seq_len=256, causal=True, capacity_factor=cf, dtype=torch.bfloat16)
    ref = P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(1), **kw)
    pip = P.ScMoEBlockPair(d, h, N, chunks=chunks,
                           generator=torch.Generator(device="cuda").manual_seed(1), **kw)
    x = torch.randn(T, d, device="cuda").bfloat16()
    with torch.no_grad():
        a, da, _ = ref(x)
        b, db, _ = pip(x)
    assert torch.equal(da.indices, db.indices) and torch.equal(da.slots, db.slots)
    assert torch.equal(a, b)


def test_chunk_routing_layout():
    from paper_2404_05019_b200 import ep, kernels as K
    T, d, N = 500, 64, 4
    x = torch.randn(T, d, device="cuda").bfloat16()
    w = torch.randn(N, d, device="cuda")
    quota = K.expert_quota(1.0, T, 2, N)
    g = K.gate_topk(x, w, 2, quota)
    dec = P.GateDecision(g.logits, g.indices, g.weights, g.dropped.bool(), g.slots, g.counts,
                         g.prob_sum, quota, quota)
    idx2, slot2, cc, rows = ep.chunk_routing(dec, 3)
    kept = g.slots < quota
    assert torch.equal((idx2 % N)[kept], g.indices[kept])
    assert torch.all(slot2[kept] < cc) and torch.all(slot2[~kept] == cc)
    # slot = chunk * cc + slot' for every kept selection
    assert torch.equal(((idx2 // N) * cc + slot2)[kept], g.slots[kept])
    assert torch.equal(rows.sum(0), dec.kept_counts())
