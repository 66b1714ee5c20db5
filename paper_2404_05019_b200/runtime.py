"""Host-buffer execution: stream batches from pinned host memory through a
module with the copies overlapped against compute.

    runner = HostStreamRunner(block)           # any module: out = f(x)[0] or f(x)
    runner.run(host_inputs, host_outputs)      # lists of pinned CPU tensors

Per step i, on three CUDA streams:

    copy-in  : H2D(input i+1)             (double-buffered device inputs)
    compute  : wait(H2D i) -> forward(i) -> record
    copy-out : wait(forward i) -> D2H(output i) into host_outputs[i]

PCIe is full duplex and both copy engines run beside the SMs, so at steady
state a step costs max(compute, H2D, D2H) instead of their sum.  Every step's
inputs are copied from host memory and every step's result is copied back;
`run` returns once the last output has landed.
"""

from __future__ import annotations

from typing import Callable, List, Optional

import torch


class CapturedStep:
    """One CUDA graph for fn(*inputs): the whole launch sequence (ctypes
    kernel launches, torch ops, memsets, autograd backward and the SGD update
    included) is recorded once and replayed with a single launch.  The path
    has no host synchronisation and static shapes, which is what makes this
    legal; inputs are copied into the graph's static buffers on replay.

        step = CapturedStep(block.train_step, [x])   # warms up, then captures
        loss = step(x_next)                            # replay
    """

    def __init__(self, fn: Callable, example_inputs, warmup: int = 3):
        self.fn = fn
        self.static_inputs = [x.clone() for x in example_inputs]
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):            # allocator warm-up off the capture stream
            for _ in range(warmup):
                fn(*self.static_inputs)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.static_output = fn(*self.static_inputs)

    def __call__(self, *inputs):
        for s, x in zip(self.static_inputs, inputs):
            if x is not s:
                s.copy_(x, non_blocking=True)
        self.graph.replay()
        return self.static_output

    def replay(self):
        self.graph.replay()
        return self.static_output


class HostStreamRunner:
    def __init__(self, fn: Callable, device: Optional[torch.device] = None):
        self.fn = fn
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.h2d = torch.cuda.Stream(device=self.device)
        self.d2h = torch.cuda.Stream(device=self.device)
        self._in = [None, None]
        self._out = [None, None]

    def _dev_buf(self, slot: int, like: torch.Tensor, which: list) -> torch.Tensor:
        b = which[slot]
        if b is None or b.shape != like.shape or b.dtype != like.dtype:
            b = torch.empty(like.shape, dtype=like.dtype, device=self.device)
            which[slot] = b
        return b

    def run(self, host_inputs: List[torch.Tensor], host_outputs: List[torch.Tensor]) -> None:
        n = len(host_inputs)
        if n == 0:
            return
        compute = torch.cuda.current_stream(self.device)
        # one callable per slot; CapturedStep slots receive the H2D directly
        # into their graph's static input and replay with a single launch
        fns = list(self.fn) if isinstance(self.fn, (list, tuple)) else [self.fn, self.fn]
        in_ready = [None] * n
        out_free = [None, None]            # D2H of the output that last used slot s
        in_free = [None, None]             # compute finished with input slot s

        def dev_in(s, like):
            if isinstance(fns[s], CapturedStep):
                return fns[s].static_inputs[0]
            return self._dev_buf(s, like, self._in)

        def issue_h2d(i):
            s = i & 1
            with torch.cuda.stream(self.h2d):
                if in_free[s] is not None:
                    self.h2d.wait_event(in_free[s])
                dev_in(s, host_inputs[i]).copy_(host_inputs[i], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.h2d)
            in_ready[i] = ev

        issue_h2d(0)
        for i in range(n):
            s = i & 1
            if i + 1 < n:
                issue_h2d(i + 1)
            compute.wait_event(in_ready[i])
            if out_free[s] is not None:
                compute.wait_event(out_free[s])   # slot s's output may be a static buffer
            f = fns[s]
            res = f.replay() if isinstance(f, CapturedStep) else f(dev_in(s, host_inputs[i]))
            out = res[0] if isinstance(res, tuple) else res
            done = torch.cuda.Event()
            done.record(compute)
            in_free[s] = done
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(done)
                if out_free[s] is not None:
                    self.d2h.wait_event(out_free[s])
                host_outputs[i].copy_(out, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.d2h)
                out_free[s] = ev
            out.record_stream(self.d2h)
        compute.wait_stream(self.d2h)
        compute.wait_stream(self.h2d)
