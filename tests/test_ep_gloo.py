"""Expert-parallel exchange over world_size 2 with the gloo backend on CPU.

The exchange code in paper_2404_05019_b200/ep.py uses only
torch.distributed, so the same functions that move the dispatch / combine
buffers over NCCL on B200s run here over gloo.  The per-rank compute is
emulated with the oracle (test side only) to check that the capacity-slotted
layout, the count exchange and the group -> local-expert mapping reproduce the
reference's moe_shared on each rank's token slice (gating.py:134-135: the
quota uses the T of the call, so per-rank results must equal the reference on
the slice).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        from paper_2404_05019_b200 import ep
        from oracle import scmoe_oracle as O

        # 1. raw exchange: buffer block (dest, e_l) tagged with (src, dest, e_l)
        E_l, C, d = 2, 3, 4
        buf = torch.zeros(world * E_l, C, d)
        for dest in range(world):
            for el in range(E_l):
                buf[dest * E_l + el] = 100 * rank + 10 * dest + el
        recv = ep.exchange_rows(buf)
        for src in range(world):
            for el in range(E_l):
                assert torch.all(recv[src * E_l + el] == 100 * src + 10 * rank + el)
        counts = torch.tensor([rank * 10 + e for e in range(world * E_l)], dtype=torch.int32)
        rc = ep.exchange_counts(counts)
        for src in range(world):
            for el in range(E_l):
                assert int(rc[src * E_l + el]) == src * 10 + rank * E_l + el

        # 2. full EP layer decomposition vs the oracle on this rank's slice
        T, d, h, N, cf = 40, 8, 16, 4, 0.75
        pp = O.init_pair(d, h, N, O.Rng(5).spawn(0), variant="scmoe", combine_mode="cg1")
        layer = pp.moe
        x = O.Rng(100 + rank).normal((T, d))
        src_x = O.Rng(200 + rank).normal((T, d))
        h_logits, _ = O.gate_logits(src_x, layer.gate)
        dec = O.standard_routing(h_logits, 1, cf)
        quota = O.expert_quota(cf, T, 1, N)
        slots = O.capacity_slots(dec.indices, N)
        disp = torch.zeros(N, quota, d, dtype=torch.float64)   # dispatch kernel semantics
        for t in range(T):
            e, s = int(dec.indices[t, 0]), int(slots[t, 0])
            if s < quota:
                disp[e, s] = torch.from_numpy(src_x[t])
        kept = torch.tensor(np.minimum(np.bincount(dec.indices[:, 0], minlength=N), quota),
                            dtype=torch.int32)
        p = ep.dispatch_exchange(disp, kept, quota)
        e_local = N // world
        y = torch.zeros_like(p.recv)
        for g in range(world * e_local):            # group g -> local expert g % E_l
            rows = int(p.recv_counts[g])
            ge = rank * e_local + g % e_local          # global expert id
            if rows:
                y[g, :rows] = torch.from_numpy(
                    O.expert_forward(p.recv[g, :rows].numpy(), layer.experts[ge]))
        back, _ = ep.combine_exchange(y)
        routed = np.zeros((T, d))
        for t in range(T):
            e, s = int(dec.indices[t, 0]), int(slots[t, 0])
            if s < quota:
                routed[t] = back[e, s].numpy()
        out = O.combine(O.expert_forward(x, layer.shared), routed, x, "cg1", layer.w_cg)
        ref, _, _ = O.moe_shared(x, layer, cf, 1, routed_src=src_x)
        np.testing.assert_allclose(out, ref, atol=1e-12)
        assert dec.dropped.any()           # the capacity path was exercised
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - surfaced through the queue
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_expert_parallel_exchange_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=170) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert results == {0: "ok", 1: "ok"}, results
