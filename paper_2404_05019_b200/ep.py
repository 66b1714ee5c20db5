"""Expert parallelism: experts sharded E/G per rank, tokens data-parallel.

Each rank routes its own T tokens with its own quota C = ceil(cf*T*k/E)
(gating.py:134-135 uses the T of the call), so per-rank results equal the
reference's moe_shared on that rank's slice.  The capacity-slotted dispatch
buffer (E, C, d) = (G, E/G, C, d) is contiguous per destination rank, so one
equal-split all-to-all moves it; a tiny int32 all-to-all carries the kept-row
counts so the grouped GEMM skips empty tiles on the device:

   dispatch buf (G, E_l, C, d) --a2a--> recv (G_src, E_l, C, d)
   grouped FFN over G*E_l groups, group (g, e) -> local expert e
   out (G_src, E_l, C, d) --a2a--> back (G, E_l, C, d) --> combine

The exchange functions only use torch.distributed, so the same code runs over
NCCL on B200 and over gloo in the CPU tests.  On a GPU they can be issued on a
side stream (`comm_stream`) to overlap the window ops chosen by sched.py.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch
import torch.distributed as dist


def exchange_counts(kept_counts: torch.Tensor, group=None) -> torch.Tensor:
    """kept_counts (E,) int32 for every global expert -> (G*E_l,) int32: the
    rows each source rank sent to each of my local experts (source-major)."""
    out = torch.empty_like(kept_counts)
    dist.all_to_all_single(out, kept_counts.contiguous(), group=group)
    return out


def exchange_rows(buf: torch.Tensor, group=None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Equal-split all-to-all of a (E, C, d) buffer laid out destination-major
    (E = G * E_l)."""
    if out is None:
        out = torch.empty_like(buf)
    dist.all_to_all_single(out.view(-1), buf.contiguous().view(-1), group=group)
    return out


@dataclass
class Pending:
    """State between the dispatch and the combine exchange of one layer."""
    recv: torch.Tensor
    recv_counts: torch.Tensor
    capacity: int
    event: Optional[torch.cuda.Event] = None


def dispatch_exchange(buf: torch.Tensor, kept_counts: torch.Tensor, capacity: int, group=None,
                      comm_stream: Optional[torch.cuda.Stream] = None) -> Pending:
    """Issue the dispatch all-to-all (on `comm_stream` if given, after the
    producer stream's current work)."""
    if comm_stream is None:
        return Pending(exchange_rows(buf, group), exchange_counts(kept_counts, group), capacity)
    producer = torch.cuda.current_stream()
    comm_stream.wait_stream(producer)
    with torch.cuda.stream(comm_stream):
        recv_counts = exchange_counts(kept_counts, group)
        recv = exchange_rows(buf, group)
        ev = torch.cuda.Event()
        ev.record(comm_stream)
    buf.record_stream(comm_stream)
    kept_counts.record_stream(comm_stream)
    return Pending(recv, recv_counts, capacity, ev)


def combine_exchange(expert_out: torch.Tensor, group=None,
                     comm_stream: Optional[torch.cuda.Stream] = None,
                     out: Optional[torch.Tensor] = None):
    """Return the expert outputs to the ranks that own the tokens; returns
    (buffer, event-or-None)."""
    if comm_stream is None:
        return exchange_rows(expert_out, group, out), None
    comm_stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(comm_stream):
        back = exchange_rows(expert_out, group, out)
        ev = torch.cuda.Event()
        ev.record(comm_stream)
    expert_out.record_stream(comm_stream)
    return back, ev


def chunk_routing(dec, n_chunks: int):
    """Chunked pipelining (distsim.py:277-300): split every expert's capacity
    C into n_chunks slices of Cc = ceil(C / n_chunks) slots and renumber
    selections into a chunk-major (n_chunks * E, Cc) buffer, so chunk c's
    dispatch / combine exchange is one contiguous (E, Cc, d) block.
    Returns (indices', slots', Cc, rows) with rows (n_chunks, E) the kept rows
    of every expert in every chunk."""
    n_exp, cap = dec.n_experts, dec.capacity
    cc = (cap + n_chunks - 1) // n_chunks
    s = dec.slots.long()
    kept = s < cap
    chunk = torch.div(s, cc, rounding_mode="floor").clamp(max=n_chunks - 1)
    idx2 = (chunk * n_exp + dec.indices.long()).to(torch.int32).contiguous()
    slot2 = torch.where(kept, s - chunk * cc, torch.full_like(s, cc)).to(torch.int32).contiguous()
    base = torch.arange(n_chunks, device=s.device)[:, None] * cc
    rows = (dec.kept_counts().long()[None, :] - base).clamp(min=0, max=cc).to(torch.int32)
    return idx2, slot2, cc, rows


def chunk_slots(dec, n_chunks: int, cc: int) -> torch.Tensor:
    """(n_chunks, T, k) int32: selection slots within chunk c (slot - c*cc) for
    the kept selections that fall in chunk c, cc (dropped) for every other —
    the per-chunk routing of the p2p dispatch, whose kernel sends only rows
    with slot < capacity."""
    s = dec.slots.long()
    kept = s < dec.capacity
    chunk = torch.div(s, cc, rounding_mode="floor")
    c = torch.arange(n_chunks, device=s.device)[:, None, None]
    mine = kept[None] & (chunk[None] == c)
    return torch.where(mine, s[None] - c * cc, torch.full_like(s[None], cc)).to(torch.int32)


def expert_parallel_ffn(experts, buf: torch.Tensor, dec, group=None) -> torch.Tensor:
    """Synchronous EP path of one layer (exchange, local grouped FFN,
    exchange back) on the current stream."""
    kept = dec.kept_counts().to(torch.int32)
    p = dispatch_exchange(buf, kept, dec.capacity, group)
    y = experts(p.recv, p.recv_counts, p.capacity)
    back, _ = combine_exchange(y, group)
    return back
