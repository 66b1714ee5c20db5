"""Memory-limited inference: routed experts held in pinned host memory
(paper App. A.3; the reference models it in scmoelab/offload.py:87-182).

The attention blocks, dense MLPs, gates and the shared expert stay resident.
Routed-expert weights live in pinned host memory, and the device keeps
S = min(N, T*k) expert slots. After the gate, the activated experts are
compacted into slots on the device.  Two migration engines:

  "copy" (default): the activated-expert list (S int32) is read back into
      pinned memory right after the gate, and the weights move as
      cudaMemcpyAsync transfers on the COPY ENGINE (scmoe_copy_rows).  No SM
      time: the transfer runs beside persistent GEMMs that hold every SM.
      The host waits for the list only once the first window op is queued,
      so the GPU never idles on the readback.
  "sm": a gather kernel (scmoe_gather_rows) pulls the rows over the host
      link; the list never leaves the GPU (no host round trip, CUDA-graph
      capturable), but the kernel needs SMs the window GEMMs occupy.

  blocking : migrate right before the expert computation, on the compute
             stream (offload.py "OffloadBlocking")
  async    : migrate on a copy stream issued at the gate point; ScMoE routes
             on the preceding representation, so the window ops (Block-MLP,
             attention, shared expert) hide the transfer and the expert
             computation waits only for the remainder (offload.py
             "OffloadAsync": stall = max(0, migration - window))

Expert outputs are bit-identical to the resident layer: same kernels, same
weights, experts renumbered into slots.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch

from . import kernels as K

MODES = ("none", "blocking", "async")


ENGINES = ("copy", "sm")


@dataclass
class SlotPlan:
    slot_idx: torch.Tensor   # (T, k) int32: selection -> device slot
    ids: torch.Tensor        # (S,) int32: expert held by slot s (first n_active valid)
    n_active: torch.Tensor   # (1,) int32 on the device
    rows: torch.Tensor       # (S,) int32 kept rows of slot s
    n_slots: int
    host: Optional[torch.Tensor] = None      # pinned (S + 1,) int32: [n_active, ids...]
    host_ev: Optional[torch.cuda.Event] = None


class ExpertOffload:
    """Host-resident copies of a RoutedExperts module plus device slots."""

    def __init__(self, experts, k_routed: int, engine: str = "copy"):
        if engine not in ENGINES:
            raise ValueError(f"unknown migration engine {engine!r}")
        self.engine = engine
        self.experts = experts
        self.k = k_routed
        self.n = experts.n_experts
        with torch.no_grad():
            self.host = [t.detach().to("cpu").contiguous().pin_memory()
                         for t in (experts.w1t, experts.b1, experts.w2t, experts.b2)]
            dev = experts.w1t.device
            # free the resident copies: peak memory = resident + S experts
            for name in ("w1t", "b1", "w2t", "b2"):
                p = getattr(experts, name)
                p.data = torch.empty(0, device=dev, dtype=p.dtype)
        self.device = dev
        self._slots = {}
        self.copy_stream = torch.cuda.Stream(device=dev)

    def host_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.host)

    def slot_buffers(self, s: int):
        b = self._slots.get(s)
        if b is None:
            b = [torch.empty((s,) + tuple(t.shape[1:]), device=self.device, dtype=t.dtype)
                 for t in self.host]
            self._slots = {s: b}          # one live size at a time
        return b

    def plan(self, dec) -> SlotPlan:
        n_tok = dec.n_tokens
        s_cnt = min(self.n, n_tok * dec.k)
        kept = dec.kept_counts()
        active = kept > 0
        slot_of = torch.cumsum(active.to(torch.int32), 0) - 1            # (N,)
        slot_of = torch.where(active, slot_of, torch.full_like(slot_of, s_cnt))
        ids = torch.zeros(s_cnt + 1, device=kept.device, dtype=torch.int32)
        ids.scatter_(0, slot_of.long(), torch.arange(self.n, device=kept.device,
                                                     dtype=torch.int32))
        rows = torch.zeros(s_cnt + 1, device=kept.device, dtype=torch.int32)
        rows.scatter_(0, slot_of.long(), kept.to(torch.int32))
        n_active = active.sum().to(torch.int32).reshape(1)
        slot_idx = slot_of[dec.indices.long()].to(torch.int32).contiguous()
        plan = SlotPlan(slot_idx, ids[:s_cnt].contiguous(), n_active, rows[:s_cnt].contiguous(),
                        s_cnt)
        if self.engine == "copy":
            # the activated-expert list to the host, queued right behind the gate
            dev_l = torch.cat([n_active, plan.ids])
            plan.host = torch.empty(s_cnt + 1, dtype=torch.int32, pin_memory=True)
            plan.host.copy_(dev_l, non_blocking=True)
        # the plan (and every earlier use of the slot buffers) is complete here:
        # the migration waits on this, not on the window ops queued after it
        plan.host_ev = torch.cuda.Event()
        plan.host_ev.record()
        return plan

    def migrate(self, plan: SlotPlan, stream=None):
        """Bring the activated experts' weights into the slots: 4 copy-engine
        transfers per run of consecutive experts ("copy": waits on the host for
        the readback of the expert list) or 4 gather kernels ("sm")."""
        bufs = self.slot_buffers(plan.n_slots)
        if self.engine == "copy":
            plan.host_ev.synchronize()
            n = int(plan.host[0])
            ids = plan.host[1:]
            for src, dst in zip(self.host, bufs):
                K.copy_rows(src, ids, n, dst, stream=stream)
            return bufs
        for src, dst in zip(self.host, bufs):
            K.gather_rows(src, plan.ids, plan.n_active, plan.n_slots, dst, stream=stream)
        return bufs

    def migrate_async(self, plan: SlotPlan):
        """Issue the migration on the copy stream after the gate; returns
        (buffers, event the expert computation must wait on)."""
        self.copy_stream.wait_event(plan.host_ev)
        with torch.cuda.stream(self.copy_stream):
            bufs = self.migrate(plan, stream=self.copy_stream)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        for t in (plan.ids, plan.n_active):
            t.record_stream(self.copy_stream)
        return bufs, ev

    def ffn(self, buf: torch.Tensor, plan: SlotPlan, bufs, capacity: int) -> torch.Tensor:
        w1t, b1, w2t, b2 = bufs
        return K.expert_ffn(buf, w1t, b1, w2t, b2, group_rows=plan.rows, rows_clip=capacity)
