"""CUDA-graph capture of whole steps (runtime.CapturedStep): the inference
forward and the training step (forward + backward through the K7 kernels +
SGD) replay bit-identically to their eager runs, and the host-streamed
runner works on graphed slots."""

import pytest
import torch

pytestmark = pytest.mark.gpu
P = R = None


def setup_module(module):
    global P, R
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2404_05019_b200 as pkg
    from paper_2404_05019_b200 import runtime
    P, R = pkg, runtime


def _block(seed, **kw):
    return P.ScMoEBlockPair(256, 512, 8, variant="scmoe", shortcut_pos="pos2", n_heads=4,
                            seq_len=256, causal=True, capacity_factor=1.25, dtype=torch.bfloat16,
                            generator=torch.Generator(device="cuda").manual_seed(seed), **kw)


def test_captured_forward_matches_eager():
    blk = _block(1)
    xs = [torch.randn(1024, 256, device="cuda").bfloat16() for _ in range(3)]

    def fwd(x):
        with torch.no_grad():
            return blk(x)[0]

    step = R.CapturedStep(fwd, [xs[0]])
    for x in xs:
        assert torch.equal(step(x).clone(), fwd(x))


def test_captured_train_step_matches_eager():
    a, b = _block(2).requires_grad_(True), _block(2).requires_grad_(True)
    x = torch.randn(1024, 256, device="cuda").bfloat16()
    tgt = torch.randn(1024, 256, device="cuda").bfloat16()
    eager = [float(a.train_step(x, lr=1e-3, target=tgt)) for _ in range(6)]
    step = R.CapturedStep(lambda x_, t_: b.train_step(x_, lr=1e-3, target=t_), [x, tgt], warmup=3)
    graphed = [float(step(x, tgt)) for _ in range(3)]
    # 3 eager warm-up steps ran before the capture (which executes nothing), so
    # replay i is step 4 + i; cuDNN's SDPA backward may accumulate dq with
    # atomics, hence the small tolerance
    assert graphed == pytest.approx(eager[3:6], rel=1e-3)
    assert torch.allclose(a.moe.experts.w1t.float(), b.moe.experts.w1t.float(), atol=1e-2)


def test_host_stream_runner_on_graphs():
    blk = _block(3)

    def fwd(x):
        with torch.no_grad():
            return blk(x)[0]

    x0 = torch.randn(1024, 256, device="cuda").bfloat16()
    steps = [R.CapturedStep(fwd, [x0]), R.CapturedStep(fwd, [x0])]
    xs = [torch.randn(1024, 256).bfloat16().pin_memory() for _ in range(5)]
    outs = [torch.empty(1024, 256, dtype=torch.bfloat16).pin_memory() for _ in range(5)]
    R.HostStreamRunner(steps).run(xs, outs)
    torch.cuda.synchronize()
    for x, o in zip(xs, outs):
        assert torch.equal(o, fwd(x.cuda()).cpu())
