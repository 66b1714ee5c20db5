"""Expert parallelism over NVLink / NVSwitch peer memory (the fused path).

The NCCL path in ep.py moves the whole capacity-padded (G, E_l, C, d)
dispatch buffer with an equal-split all-to-all, then moves the expert outputs
back the same way.  Here the kernels do the transfers themselves
(csrc/dispatch.cu, K9/K10):

    gate (compute) --> scmoe_ep_dispatch_p2p (side stream, bounded grid):
                       kept rows stored into recv on their owner rank,
                       counts published, epoch flag released on every peer
    owner: scmoe_ep_wait(0) -> grouped FFN recv -> y -> scmoe_ep_signal(1)
    source: scmoe_ep_wait(1) -> scmoe_ep_combine_p2p: expert rows read from
            y on their owner, fused with SE, combination gate and residual

Only kept rows cross NVLink (no padding, no staging copy), the dispatch copy
runs beside the window ops on a side stream, and the return trip is folded
into the combine kernel's loads.  Ordering is carried by per-rank epoch
counters in device memory, so a captured CUDA graph replays correctly.

`PeerExchange.from_group` maps every rank's buffers into every peer with
CUDA IPC handles exchanged over the process group (or torch symmetric
memory) — allocation and handle exchange only; every byte of the exchange is
moved by our kernels.  `PeerExchange.virtual` lays out G ranks'
buffers on ONE GPU with the same pointer tables, so the exchange logic is
tested bit-for-bit on a single B200.

Buffer reuse across calls is safe by construction: a source's next dispatch
is issued after its combine, which waited for every owner's y-ready flag of
the previous call (so the owners are done reading recv); an owner's next FFN
waits for every source's next dispatch, issued after that source's combine
finished reading y.
"""

from __future__ import annotations

from typing import List, Optional

import torch

from . import _lib
from ._lib import check, dtype_code, lib, ptr, stream_ptr


class PeerExchange:
    """Receive / output buffers, counts, flags and peer tables of one rank."""

    def __init__(self, world: int, rank: int, e_local: int, capacity: int, d_model: int,
                 dtype: torch.dtype, device, storage: Optional[torch.Tensor] = None,
                 chunks: int = 1):
        """capacity: slots per expert of ONE chunk.  chunks > 1 (chunked
        pipelining, distsim.py:277-300): `chunks` independent exchanges, each
        with its own recv / y rows, counts, flags and epoch counter, whose
        `back` rows are contiguous chunk-major, (chunks * E, capacity, d) — the
        layout ep.chunk_routing numbers selections in, so one combine gathers
        every chunk."""
        if chunks < 1:
            raise ValueError("chunks must be >= 1")
        self.world, self.rank, self.e_local = world, rank, e_local
        self.capacity, self.d_model, self.dtype = capacity, d_model, dtype
        self.chunks = chunks
        dev = torch.device(device)
        G = world * e_local
        self._sizes, self._offs, off = self.layout(world, e_local, capacity, d_model, dtype, chunks)
        self.nbytes = off
        if storage is None:
            storage = torch.zeros(off, dtype=torch.uint8, device=dev)
        if storage.numel() < off:
            raise ValueError("peer storage too small")
        self.storage = storage
        b = storage
        def part(i):
            return b[self._offs[i]:self._offs[i] + self._sizes[i]]
        # chunk c of a (chunks * G, capacity, d) buffer: rows [c*G, (c+1)*G)
        self.recv = part(0).view(dtype).view(chunks * G, capacity, d_model)
        self.y = part(1).view(dtype).view(chunks * G, capacity, d_model)
        self.back = part(2).view(dtype).view(chunks * G, capacity, d_model)
        self.recv_counts = part(3).view(torch.int32)              # (chunks * G,)
        self.flags = part(4).view(torch.int32)                    # (chunks, 2, world)
        self.epoch = torch.zeros(4 * chunks, dtype=torch.int32, device=dev)
        self.tables = None

    @staticmethod
    def layout(world, e_local, capacity, d_model, dtype, chunks: int = 1):
        """(sizes, offsets, total bytes) of [recv | y | back | recv_counts |
        flags], each 256-byte aligned, each holding `chunks` consecutive
        per-chunk parts."""
        G = world * e_local
        esz = torch.tensor([], dtype=dtype).element_size()
        rows = G * capacity * d_model
        sizes = [chunks * n for n in (rows * esz, rows * esz, rows * esz, G * 4, 2 * world * 4)]
        offs, off = [], 0
        for n in sizes:
            offs.append(off)
            off += (n + 255) // 256 * 256
        return sizes, offs, off

    def _chunk_stride(self, i: int) -> int:
        """Bytes between consecutive chunks' parts of region i."""
        return self._sizes[i] // self.chunks

    def part(self, name: str, chunk: int = 0) -> torch.Tensor:
        """Chunk `chunk` of recv / y / back ((G, capacity, d)) or recv_counts."""
        G = self.world * self.e_local
        if name == "recv_counts":
            return self.recv_counts[chunk * G:(chunk + 1) * G]
        return getattr(self, name)[chunk * G:(chunk + 1) * G]

    # -- peer tables -------------------------------------------------------------
    def set_peer_bases(self, bases: List[int]) -> "PeerExchange":
        """bases[r] = address of rank r's storage as mapped in THIS process."""
        if len(bases) != self.world:
            raise ValueError("one base per rank")
        dev = self.storage.device
        # tables[c][i][r]: region i (recv, y, back, recv_counts, flags) of
        # chunk c on rank r
        tab = torch.tensor([[[b + o + c * self._chunk_stride(i) for b in bases]
                             for i, o in enumerate(self._offs)] for c in range(self.chunks)],
                           dtype=torch.int64, device=dev)
        self.tables = tab
        # fused return: group (src, el) of this owner -> the source's back rows
        # (rank * E_l + el) * C (global expert order on the source), per chunk
        esz = torch.tensor([], dtype=self.dtype).element_size()
        row = self.capacity * self.d_model * esz
        G = self.world * self.e_local
        self.group_out = torch.tensor(
            [[bases[g // self.e_local] + self._offs[2] + c * self._chunk_stride(2) +
              (self.rank * self.e_local + g % self.e_local) * row for g in range(G)]
             for c in range(self.chunks)], dtype=torch.int64, device=dev)
        return self

    def _tab(self, i: int, chunk: int = 0) -> int:
        return self.tables[chunk, i].data_ptr()

    def _flags(self, chunk: int) -> int:
        return self.flags[chunk * 2 * self.world:].data_ptr()

    def _epoch(self, chunk: int) -> int:
        return self.epoch[4 * chunk:].data_ptr()

    @classmethod
    def virtual(cls, world: int, e_local: int, capacity: int, d_model: int, dtype, device,
                chunks: int = 1):
        """`world` ranks on one GPU: separate storages, peer tables pointing at
        each other's storage — the same addressing the NVLink path uses."""
        xs = [cls(world, r, e_local, capacity, d_model, dtype, device, chunks=chunks)
              for r in range(world)]
        bases = [x.storage.data_ptr() for x in xs]
        for x in xs:
            x.set_peer_bases(bases)
        return xs

    @classmethod
    def from_group(cls, group, e_local: int, capacity: int, d_model: int, dtype, device,
                   method: str = "auto", chunks: int = 1):
        """Peer-mapped storage over a process group.  Allocation and handle
        exchange only — every byte of the exchange is moved by our kernels.

        method "ipc": each rank allocates its storage, the CUDA IPC handles
        (torch's storage sharing: cudaIpcGetMemHandle / cudaIpcOpenMemHandle
        with lazy peer access) travel through the group as objects, and every
        rank maps every peer's storage.  Works across the GPUs of a node
        (NVLink peer access) and across processes sharing one GPU.
        method "symm": torch symmetric memory (one GPU per rank only; one
        mapping per peer without a CUDA context per peer device).
        method "auto": "symm" when every rank can rendezvous, else "ipc"
        (e.g. ranks sharing a GPU).  The choice is agreed over the group."""
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        if method == "auto":
            ok = 1
            try:
                import torch.distributed._symmetric_memory  # noqa: F401
            except Exception:
                ok = 0
            flags = [None] * world
            dist.all_gather_object(flags, ok, group=group)
            if all(flags):
                try:
                    x = cls.from_group(group, e_local, capacity, d_model, dtype, device,
                                       method="symm", chunks=chunks)
                    ok = 1
                except Exception:   # e.g. two ranks on one device
                    x, ok = None, 0
                dist.all_gather_object(flags, ok, group=group)
                if all(flags):      # every rank mapped every peer: agreed
                    return x
            method = "ipc"
        if method == "symm":
            import torch.distributed._symmetric_memory as symm_mem
            nbytes = cls.layout(world, e_local, capacity, d_model, dtype, chunks)[2]
            name = group.group_name if hasattr(group, "group_name") else group
            buf = symm_mem.empty(nbytes, dtype=torch.uint8, device=device)
            buf.zero_()
            hdl = symm_mem.rendezvous(buf, name)
            own = buf.data_ptr() - hdl.buffer_ptrs[rank]
            bases = [p + own for p in hdl.buffer_ptrs]
            x = cls(world, rank, e_local, capacity, d_model, dtype, device, storage=buf,
                    chunks=chunks)
            x._handle = hdl
            hdl.barrier()
            return x.set_peer_bases(bases)
        if method != "ipc":
            raise ValueError(f"unknown method {method!r}")
        x = cls(world, rank, e_local, capacity, d_model, dtype, device, chunks=chunks)
        torch.cuda.synchronize()             # storage zeroed before peers map it
        meta = x.storage.untyped_storage()._share_cuda_()
        metas = [None] * world
        dist.all_gather_object(metas, meta, group=group)
        x._peer_storages = []
        bases = []
        for r, m in enumerate(metas):
            if r == rank:
                bases.append(x.storage.data_ptr())
            else:
                st = torch.UntypedStorage._new_shared_cuda(*m)
                x._peer_storages.append(st)
                bases.append(st.data_ptr())
        dist.barrier(group=group)            # every rank mapped every peer
        return x.set_peer_bases(bases)

    # -- the exchange ------------------------------------------------------------
    # `chunk` selects one of the `chunks` independent exchanges (0 when
    # unchunked); each has its own flags and epoch, so chunk c's expert can
    # start as soon as chunk c's rows landed, while chunk c+1 is in flight.
    def dispatch(self, x: torch.Tensor, indices: torch.Tensor, slots: torch.Tensor,
                 counts: torch.Tensor, max_ctas: int = 0, stream=None, chunk: int = 0) -> None:
        """Kept rows (slot < capacity) to their owners' recv rows of `chunk`;
        counts (E,) per global expert (kept = min(count, capacity))."""
        T, d = x.shape
        k = indices.shape[1]
        check(lib().scmoe_ep_dispatch_p2p(
            ptr(x), dtype_code(x.dtype), x.stride(0), T, d, k, ptr(indices), ptr(slots),
            ptr(counts), self.capacity, self.world, self.rank, self.e_local, self._tab(0, chunk),
            self._tab(3, chunk), self._tab(4, chunk), self._epoch(chunk), max_ctas,
            stream_ptr(stream)))

    def wait(self, which: int, stream=None, chunk: int = 0) -> None:
        check(lib().scmoe_ep_wait(self._flags(chunk), which, self.world, self._epoch(chunk),
                                  stream_ptr(stream)))

    def signal(self, which: int, stream=None, chunk: int = 0) -> None:
        check(lib().scmoe_ep_signal(self._tab(4, chunk), which, self.world, self.rank,
                                    self._epoch(chunk), stream_ptr(stream)))

    def expert_ffn(self, experts, signal: bool = True, stream=None, chunk: int = 0) -> torch.Tensor:
        """Owner side: wait for every source's rows, grouped FFN recv -> y
        (groups (src, el) -> local expert el); with `signal`, release y-ready
        for the pull-form combine."""
        self.wait(0, stream, chunk)
        y = self.part("y", chunk)
        experts(self.part("recv", chunk), self.part("recv_counts", chunk), self.capacity, out=y,
                stream=stream)
        if signal:
            self.signal(1, stream, chunk)
        return y

    def expert_ffn_to_peers(self, experts, stream=None, chunk: int = 0) -> None:
        """Owner side, fused form of the return trip: wait for every source's
        rows, then one grouped FFN whose GEMM2 epilogue stores each finished
        row tile straight into the source's `back` buffer over peer memory
        (no local y, no separate return kernel); then release flag 1."""
        self.wait(0, stream, chunk)
        check(lib().scmoe_expert_ffn_to_peers(
            ptr(self.part("recv", chunk)), dtype_code(self.dtype), ptr(experts.w1t),
            ptr(experts.b1), ptr(experts.w2t), ptr(experts.b2), ptr(self._hidden(experts)),
            self.group_out[chunk].data_ptr(), self.world * self.e_local, experts.n_experts,
            self.capacity, ptr(self.part("recv_counts", chunk)), self.capacity, self.d_model,
            experts.d_hidden, stream_ptr(stream)))
        self.signal(1, stream, chunk)

    def _hidden(self, experts) -> torch.Tensor:
        h = getattr(self, "_hidden_buf", None)
        shape = (self.world * self.e_local, self.capacity, experts.d_hidden)
        if h is None or tuple(h.shape) != shape:
            h = torch.empty(shape, dtype=self.dtype, device=self.recv.device)
            self._hidden_buf = h
        return h

    def push_back(self, max_ctas: int = 0, stream=None, chunk: int = 0) -> None:
        """Owner side, push form of the return trip: valid rows of y into every
        source's `back` buffer, then release flag 1 on the sources."""
        check(lib().scmoe_ep_return_p2p(
            ptr(self.part("y", chunk)), dtype_code(self.dtype),
            ptr(self.part("recv_counts", chunk)), self.capacity, self.d_model, self.world,
            self.rank, self.e_local, self._tab(2, chunk), self._tab(4, chunk),
            self._epoch(chunk), max_ctas, stream_ptr(stream)))

    def combine_local(self, indices, slots, weights, **kw) -> torch.Tensor:
        """Source side after the return trip: wait for every owner's rows of
        every chunk, then the ordinary combine over `back` ((chunks * E, C, d),
        global expert order; chunked callers pass ep.chunk_routing's chunk-
        major indices / slots)."""
        from . import kernels as K
        stream = kw.pop("stream", None)
        for c in range(self.chunks):
            self.wait(1, stream, c)
        return K.combine(self.back.view(-1, self.capacity, self.d_model), indices, slots, weights,
                         self.capacity, stream=stream, **kw)

    def combine(self, indices, slots, weights, se_out=None, mode: str = "direct_add",
                x_cur=None, w_cg=None, residual=None, out=None, stream=None) -> torch.Tensor:
        """Source side: wait for every owner's y, then the fused gather-sum
        (unchunked exchanges)."""
        if self.chunks != 1:
            raise ValueError("the pull-form combine reads one chunk's y; use combine_local")
        self.wait(1, stream)
        T, k = indices.shape
        if out is None:
            out = torch.empty(T, self.d_model, dtype=self.dtype, device=indices.device)
        check(lib().scmoe_ep_combine_p2p(
            ptr(se_out), self._tab(1), ptr(x_cur), ptr(w_cg), _lib.COMBINE_MODES[mode],
            ptr(residual), ptr(indices), ptr(slots), ptr(weights), self.capacity, T,
            self.d_model, k, dtype_code(self.dtype), self.world, self.rank, self.e_local,
            ptr(out), stream_ptr(stream)))
        return out
