"""Memory-limited inference: routed experts held in pinned host memory
(paper App. A.3; the reference models it in scmoelab/offload.py:87-182).

The attention blocks, dense MLPs, gates and the shared expert stay resident.
Routed-expert weights live in pinned host memory, and the device keeps
S = min(N, T*k) expert slots. After the gate, the activated experts are
compacted into slots on the device, and a gather kernel (scmoe_gather_rows)
pulls their weights over the host link straight from the pinned buffers. The
activated-expert list never leaves the GPU, so there is no host round trip.

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

import torch

from . import kernels as K

MODES = ("none", "blocking", "async")


@dataclass
class SlotPlan:
    slot_idx: torch.Tensor   # (T, k) int32: selection -> device slot
    ids: torch.Tensor        # (S,) int32: expert held by slot s (first n_active valid)
    n_active: torch.Tensor   # (1,) int32 on the device
    rows: torch.Tensor       # (S,) int32 kept rows of slot s
    n_slots: int


class ExpertOffload:
    """Host-resident copies of a RoutedExperts module plus device slots."""

    def __init__(self, experts, k_routed: int):
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
        return SlotPlan(slot_idx, ids[:s_cnt].contiguous(), n_active, rows[:s_cnt].contiguous(),
                        s_cnt)

    def migrate(self, plan: SlotPlan, stream=None):
        """Pull the activated experts' weights into the slots (4 gathers)."""
        bufs = self.slot_buffers(plan.n_slots)
        for src, dst in zip(self.host, bufs):
            K.gather_rows(src, plan.ids, plan.n_active, plan.n_slots, dst, stream=stream)
        return bufs

    def migrate_async(self, plan: SlotPlan):
        """Issue the migration on the copy stream after the gate; returns
        (buffers, event the expert computation must wait on)."""
        cur = torch.cuda.current_stream(self.device)
        self.copy_stream.wait_stream(cur)
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
