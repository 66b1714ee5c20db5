"""Memory-limited inference (offload.py; reference scmoelab/offload.py:87-182):
with the routed experts in pinned host memory, only the activated experts
migrate into device slots, and the block output must equal the resident
block's bit for bit in both modes ("blocking" = OffloadBlocking, "async" =
OffloadAsync started at the shortcut gate point)."""

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


def _pair(variant, k, cf, d=256, h=512, N=8, seed=3):
    kw = dict(variant=variant, k_routed=k, shortcut_pos="pos2" if variant == "scmoe" else None,
              n_heads=4, seq_len=None, causal=False, capacity_factor=cf, dtype=torch.bfloat16)
    return P.ScMoEBlockPair(d, h, N, generator=torch.Generator(device="cuda").manual_seed(seed),
                            **kw)


def test_gather_rows_from_pinned_host():
    from paper_2404_05019_b200 import kernels as K
    src = torch.randn(12, 33, 40).bfloat16().pin_memory()
    ids = torch.tensor([7, 2, 11, 0, 5], device="cuda", dtype=torch.int32)
    n = torch.tensor([3], device="cuda", dtype=torch.int32)
    out = torch.full((5, 33, 40), 7.0, device="cuda").bfloat16()
    K.gather_rows(src, ids, n, 5, out)
    torch.cuda.synchronize()
    ref = src[ids.cpu().long()].cuda()
    assert torch.equal(out[:3], ref[:3])
    assert torch.all(out[3:] == 7.0)          # rows past n_rows are untouched
    # device-resident sources go through the same kernel
    out2 = torch.zeros(5, 33, 40, device="cuda").bfloat16()
    K.gather_rows(src.cuda(), ids, torch.tensor([5], device="cuda", dtype=torch.int32), 5, out2)
    assert torch.equal(out2, ref)
    with pytest.raises(ValueError):
        K.gather_rows(torch.randn(4, 8).bfloat16(), ids[:1], n, 1,
                      torch.empty(1, 8, device="cuda").bfloat16())


def test_copy_rows_copy_engine():
    """scmoe_copy_rows: host-known row ids, cudaMemcpyAsync per run of
    consecutive ids (copy engine, no kernel)."""
    from paper_2404_05019_b200 import kernels as K
    src = torch.randn(12, 33, 40).bfloat16().pin_memory()
    ids = torch.tensor([7, 8, 9, 2, 11, 0, 5], dtype=torch.int32)
    out = torch.full((7, 33, 40), 7.0, device="cuda").bfloat16()
    K.copy_rows(src, ids, 5, out)
    torch.cuda.synchronize()
    assert torch.equal(out[:5].cpu(), src[ids[:5].long()])
    assert torch.all(out[5:] == 7.0)
    K.copy_rows(src.cuda(), ids, 7, out)          # device sources too
    assert torch.equal(out.cpu(), src[ids.long()])
    with pytest.raises(ValueError):
        K.copy_rows(src, ids.cuda(), 1, out)       # ids must be on the host
    with pytest.raises(ValueError):
        K.copy_rows(src, ids, 8, out)


@pytest.mark.parametrize("variant,k,cf", [("scmoe", 1, 1.25), ("standard", 2, 1.0),
                                          ("shared", 2, 0.5)])
@pytest.mark.parametrize("mode", ["blocking", "async"])
@pytest.mark.parametrize("engine", ["copy", "sm"])
@pytest.mark.parametrize("T", [3, 64, 1024])
def test_offload_equals_resident(variant, k, cf, mode, engine, T):
    ref = _pair(variant, k, cf)
    off = _pair(variant, k, cf).enable_offload(mode, engine)
    assert off.offload.host_bytes() > 0
    x = torch.randn(T, 256, device="cuda").bfloat16()
    with torch.no_grad():
        a, da, _ = ref(x)
        for _ in range(2):            # second call reuses the slot buffers
            b, db, _ = off(x)
    torch.cuda.synchronize()
    assert torch.equal(da.indices, db.indices) and torch.equal(da.slots, db.slots)
    assert torch.equal(a, b)


def test_offload_frees_and_bounds_device_memory():
    torch.cuda.synchronize()
    N, d, h = 16, 512, 2048
    blk = _pair("scmoe", 1, 1.0, d=d, h=h, N=N)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    blk.enable_offload("async")
    torch.cuda.synchronize()
    freed = before - torch.cuda.memory_allocated()
    expert_bytes = N * (2 * d * h + d + h) * 2
    assert freed >= expert_bytes * 0.99
    # a 2-token step holds at most 2 experts on the device
    x = torch.randn(2, d, device="cuda").bfloat16()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    with torch.no_grad():
        blk(x)
    torch.cuda.synchronize()
    assert torch.cuda.max_memory_allocated() - base < 3 * expert_bytes / N


def test_offload_rejects_training_modes():
    blk = _pair("scmoe", 1, 1.0)
    with pytest.raises(P.ConfigError):
        blk.enable_offload("sometimes")
    blk.enable_offload("blocking")
    blk.chunks = 2
    with pytest.raises(NotImplementedError):
        with torch.no_grad():
            blk(torch.randn(8, 256, device="cuda").bfloat16())
