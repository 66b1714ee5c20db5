"""Device timelines: CUDA-event spans per op and stream, and the overlap metric.

`comm_overlap_fraction` has the semantics of the reference's metric
(scmoelab/distsim.py:456-469): the share of all-to-all time covered by the
union of compute spans; 1.0 when there is no communication.  Spans come from
CUDA events recorded on the stream each op runs on, after its cross-stream
waits, so the numbers are device time, not host wall clock.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import torch

COMM_KINDS = ("dispatch", "combine")


@dataclass
class Span:
    op: str
    stream: str          # "compute" | "comm"
    start_ms: float
    end_ms: float

    @property
    def ms(self) -> float:
        return self.end_ms - self.start_ms


def _union(intervals: Sequence[Tuple[float, float]]) -> List[Tuple[float, float]]:
    merged: List[List[float]] = []
    for a, b in sorted(intervals):
        if merged and a <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], b)
        else:
            merged.append([a, b])
    return [(a, b) for a, b in merged]


def comm_overlap_fraction(spans: Sequence[Span]) -> float:
    compute = _union([(s.start_ms, s.end_ms) for s in spans if s.stream != "comm"])
    total = hidden = 0.0
    for s in spans:
        if s.stream != "comm":
            continue
        total += s.ms
        for a, b in compute:
            hidden += max(0.0, min(b, s.end_ms) - max(a, s.start_ms))
    return 1.0 if total == 0.0 else hidden / total


def exposed_comm_ms(spans: Sequence[Span]) -> float:
    comm = sum(s.ms for s in spans if s.stream == "comm")
    return comm * (1.0 - comm_overlap_fraction(spans))


def window_makespan_ms(spans: Sequence[Span], window_ops: Sequence[str]) -> float:
    """Measured counterpart of sched.slot_makespan: device time from the
    first start to the last end of the overlap window's ops, the routed
    expert and both exchanges (max(pre, t_disp) + t_expert + max(post,
    t_comb) when the schedule is realised exactly)."""
    names = set(window_ops) | {"expert"} | set(COMM_KINDS)
    sel = [s for s in spans if s.op in names]
    if not sel:
        return 0.0
    return max(s.end_ms for s in sel) - min(s.start_ms for s in sel)


def kernel_overlap(intervals, is_comm, is_idle=lambda name: False):
    """comm_overlap_fraction on KERNEL EXECUTION intervals (CUPTI start / end
    of every kernel of one step, same device clock): the share of the
    exchange kernels' execution time during which a compute kernel was also
    executing.  Unlike the event spans, a comm kernel queued behind a grid
    that holds every SM does not count as hidden.  `is_idle` drops kernels
    that only wait (the flag-spin waits on the compute stream).
    intervals: [(name, start_us, end_us)].  Returns (fraction, comm_us,
    exposed_us)."""
    comp = _union([(a, b) for n, a, b in intervals if not is_comm(n) and not is_idle(n)])
    total = hidden = 0.0
    for n, a, b in intervals:
        if not is_comm(n):
            continue
        total += b - a
        for x, y in comp:
            hidden += max(0.0, min(y, b) - max(x, a))
    frac = 1.0 if total == 0.0 else hidden / total
    return frac, total, total - hidden


class Recorder:
    """Records (start, end) event pairs per op; `spans()` syncs once."""

    def __init__(self, enabled: bool = True):
        self.enabled = enabled
        self._events: List[Tuple[str, str, torch.cuda.Event, torch.cuda.Event]] = []
        self._base: Optional[torch.cuda.Event] = None

    def begin(self, stream: torch.cuda.Stream):
        if not self.enabled:
            return
        self._base = torch.cuda.Event(enable_timing=True)
        self._base.record(stream)

    def op(self, name: str, kind: str, stream: torch.cuda.Stream):
        rec = self

        class _Ctx:
            def __enter__(self_inner):
                if rec.enabled:
                    self_inner.s = torch.cuda.Event(enable_timing=True)
                    self_inner.s.record(stream)
                return self_inner

            def __exit__(self_inner, *exc):
                if rec.enabled:
                    e = torch.cuda.Event(enable_timing=True)
                    e.record(stream)
                    rec._events.append((name, kind, self_inner.s, e))
                return False

        return _Ctx()

    def spans(self) -> List[Span]:
        if not self.enabled or self._base is None:
            return []
        torch.cuda.synchronize()
        out = [Span(n, k, self._base.elapsed_time(s), self._base.elapsed_time(e))
               for n, k, s, e in self._events]
        return sorted(out, key=lambda s: (s.start_ms, s.end_ms, s.op))

    def durations(self) -> Dict[str, float]:
        d: Dict[str, float] = {}
        for s in self.spans():
            d[s.op] = d.get(s.op, 0.0) + s.ms
        return d
