"""Generate the golden vectors that pin the oracle to the REAL reference.

Run in the dev container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package `scmoelab` from
/root/reference/pkg/src and records its outputs for the hot-path functions:
gating (select_topk / apply_capacity / expert_quota / load_balance_loss,
gating.py:93-170), the layer entries (moe_shared / moe_standard,
arch.py:463-504), the block-pair wiring (arch.model_forward, arch.py:553-631),
the scheduler (sched.choose_slot, sched.py:88-98) and the overlap metric
(distsim.comm_overlap_fraction, distsim.py:456-469).  Outputs are written as
compressed .npz / .json next to this script.  Nothing on the GPU box reads
/root/reference; only these committed files travel.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import scmoelab  # noqa: F401
    from scmoelab import arch, distsim, gating, sched
    from scmoelab.numkit import Rng
    return arch, distsim, gating, sched, Rng


def gating_cases(gating, Rng):
    out = {}
    rng = np.random.default_rng(20251017)
    cases = []
    for i in range(300):
        t = int(rng.integers(1, 48))
        n = int(rng.integers(1, 17))
        k = int(rng.integers(1, min(n, 4) + 1))
        cf = float(rng.uniform(0.25, 3.0))
        h = rng.standard_normal((t, n))
        mode = i % 4
        if mode == 1:      # coarse grid -> many exact ties
            h = np.round(h * 2.0) / 2.0
        elif mode == 2:    # signed zeros and duplicated maxima
            h = np.round(h)
            h[rng.random(h.shape) < 0.3] = -0.0
            h[rng.random(h.shape) < 0.3] = 0.0
        elif mode == 3:    # whole rows tied
            h[rng.random(t) < 0.5] = 0.25
        h = h.astype(np.float32).astype(np.float64)   # "identical fp32 logits"
        dec = gating.select_topk(h, k)
        cap = gating.CapacityConfig(cf)
        capped = gating.apply_capacity(dec, cap, n, t)
        cases.append(dict(t=t, n=n, k=k, cf=cf,
                          quota=gating.expert_quota(cap, t, k, n),
                          lb=gating.load_balance_loss(capped, n)))
        out[f"g{i}_h"] = h
        out[f"g{i}_idx"] = capped.indices.astype(np.int64)
        out[f"g{i}_w"] = capped.weights
        out[f"g{i}_drop"] = capped.dropped
    # larger cases with heavy dropping (cf = 1.0 and below)
    for j, (t, n, k, cf) in enumerate([(4096, 8, 1, 1.0), (4096, 8, 2, 1.0),
                                       (3000, 16, 2, 0.5), (2048, 4, 1, 0.75)]):
        i = 300 + j
        h = (rng.standard_normal((t, n)) + np.linspace(0, 1.5, n)[None, :])
        h = h.astype(np.float32).astype(np.float64)
        cap = gating.CapacityConfig(cf)
        capped = gating.apply_capacity(gating.select_topk(h, k), cap, n, t)
        cases.append(dict(t=t, n=n, k=k, cf=cf, quota=gating.expert_quota(cap, t, k, n),
                          lb=gating.load_balance_loss(capped, n)))
        out[f"g{i}_h"] = h
        out[f"g{i}_idx"] = capped.indices.astype(np.int64)
        out[f"g{i}_w"] = capped.weights
        out[f"g{i}_drop"] = capped.dropped
    np.savez_compressed(os.path.join(HERE, "gating_cases.npz"), **out)
    with open(os.path.join(HERE, "gating_cases.json"), "w") as fh:
        json.dump(cases, fh, indent=0)


def _flatten_layer(prefix, layer, out):
    for e_i, e in enumerate(layer.experts):
        for nm in ("w1", "b1", "w2", "b2"):
            out[f"{prefix}e{e_i}_{nm}"] = getattr(e, nm)
    if layer.shared is not None:
        for nm in ("w1", "b1", "w2", "b2"):
            out[f"{prefix}se_{nm}"] = getattr(layer.shared, nm)
    out[f"{prefix}wg"] = layer.gate.w_gate
    out[f"{prefix}wn"] = layer.gate.w_noise
    if layer.combine.w_cg is not None:
        out[f"{prefix}wcg"] = layer.combine.w_cg


def layer_and_pair_cases(arch, Rng):
    """moe_shared / moe_standard on init_params weights + block-pair forwards."""
    out, meta = {}, []
    combos = []
    for comb in ("direct_add", "cg1", "cg2"):
        for pos in ("pos1", "pos2", "pos3"):
            combos.append(dict(variant="scmoe", shortcut_pos=pos, combine_mode=comb, k_routed=1))
        combos.append(dict(variant="shared", combine_mode=comb, k_routed=1))
    combos.append(dict(variant="scmoe", shortcut_pos="pos2", combine_mode="direct_add", k_routed=2))
    combos.append(dict(variant="standard", k_routed=2))
    combos.append(dict(variant="standard", k_routed=1))
    combos.append(dict(variant="scmoe", shortcut_pos="pos2", combine_mode="cg1",
                       k_routed=1, noise_enabled=True))
    combos.append(dict(variant="scmoe", shortcut_pos="pos1", combine_mode="direct_add",
                       k_routed=1, pre_layernorm=True))
    combos.append(dict(variant="dgmoe", shortcut_pos="pos2", k_routed=1))
    combos.append(dict(variant="dgmoe", shortcut_pos="pos2", k_routed=1, dgmoe_constraint=False))
    for i, kw in enumerate(combos):
        t, d, h, n = 24, 8, 16, 4
        cf = [2.0, 1.0, 0.5][i % 3]
        cfg = arch.ModelConfig(n_blocks=2, d_model=d, d_hidden=h, n_experts=n,
                               capacity_factor=cf, **kw)
        rng = Rng(100 + i)
        params = arch.init_params(cfg, rng.spawn(0))
        tokens = rng.spawn(1).normal((t, d))
        noise_rng = Rng(7) if cfg.noise_enabled else None
        res = arch.model_forward(cfg, params, tokens, rng=noise_rng)
        m = res.trace.moe[0]
        p = f"c{i}_"
        if m.decision_prev is not None:
            out[p + "idx_prev"] = m.decision_prev.indices.astype(np.int64)
            out[p + "drop_prev"] = m.decision_prev.dropped
            out[p + "out"] = np.asarray(res.output)
            out[p + "idx"] = m.decision.indices.astype(np.int64)
            out[p + "drop"] = m.decision.dropped
            out[p + "tokens"] = tokens
            out[p + "aux"] = np.asarray(m.aux_loss)
            meta.append(dict(t=t, d=d, h=h, n=n, cf=cf, seed=100 + i, **kw))
            continue
        out[p + "tokens"] = tokens
        out[p + "out"] = np.asarray(res.output)
        out[p + "idx"] = m.decision.indices.astype(np.int64)
        out[p + "drop"] = m.decision.dropped
        out[p + "w"] = m.decision.weights
        out[p + "logits"] = m.decision.logits
        if m.decision.eps is not None:
            out[p + "eps"] = m.decision.eps
        out[p + "src"] = m.routed_input
        out[p + "xcur"] = m.current_input
        # the layer entry alone, on the recorded inputs (replaying the noise)
        layer = params.blocks[1].feed
        replay = arch.MoEReplay(eps=m.decision.eps)
        if cfg.variant == "standard":
            lo, ldec, laux = arch.moe_standard(m.current_input, layer, cfg.capacity(),
                                               cfg.k_routed, replay=replay)
        else:
            src = m.routed_input if cfg.variant == "scmoe" else None
            lo, ldec, laux = arch.moe_shared(m.current_input, layer, cfg.capacity(),
                                             cfg.k_routed, replay=replay, routed_src=src)
        out[p + "layer_out"] = np.asarray(lo)
        out[p + "aux"] = np.asarray(float(np.asarray(laux).reshape(())))
        # raw init_params arrays of block 0 + block 1 to pin the init order
        b0, b1 = params.blocks
        for nm in ("w_q", "w_k", "w_v", "w_o"):
            out[p + "a0_" + nm] = getattr(b0.attn, nm)
            out[p + "a1_" + nm] = getattr(b1.attn, nm)
        for nm in ("w1", "b1", "w2", "b2"):
            out[p + "mlp_" + nm] = getattr(b0.feed, nm)
        _flatten_layer(p + "L_", b1.feed, out)
        meta.append(dict(t=t, d=d, h=h, n=n, cf=cf, seed=100 + i, **kw))
    np.savez_compressed(os.path.join(HERE, "layer_cases.npz"), **out)
    with open(os.path.join(HERE, "layer_cases.json"), "w") as fh:
        json.dump(meta, fh, indent=0)


def cfg1_case(arch, Rng):
    """BASELINE configs[0]: d=256, h=1024 (4d), N=8, top-1 + SE, cf 1.0, pos2,
    4x128 = 512 tokens, fp64 reference.  Stored compactly (decision + first
    rows + row sums) — the oracle recomputes the rest from the seed."""
    cfg = arch.ModelConfig(n_blocks=2, d_model=256, d_hidden=1024, n_experts=8,
                           k_routed=1, variant="scmoe", shortcut_pos="pos2",
                           capacity_factor=1.0)
    rng = Rng(0)
    params = arch.init_params(cfg, rng.spawn(0))
    tokens = rng.spawn(1).normal((512, 256))
    out, trace = arch.forward(cfg, params, tokens)
    m = trace.moe[0]
    np.savez_compressed(os.path.join(HERE, "cfg1_case.npz"),
                        out_head=out[:16], out_rowsum=out.sum(axis=1),
                        idx=m.decision.indices.astype(np.int64), drop=m.decision.dropped,
                        aux=np.asarray(m.aux_loss), wg_head=params.blocks[1].feed.gate.w_gate[:4])


def sched_cases(sched, distsim):
    rng = np.random.default_rng(4)
    vecs = []
    for _ in range(400):
        m = int(rng.integers(1, 7))
        comp = [float(v) / 4.0 for v in rng.integers(0, 400, m)]
        c = sched.CostVector(comp=comp, t_disp=float(rng.integers(0, 400)) / 4.0,
                             t_comb=float(rng.integers(0, 400)) / 4.0,
                             t_expert=float(rng.integers(0, 160)) / 4.0)
        ch = sched.choose_slot(c)
        vecs.append(dict(comp=comp, t_disp=c.t_disp, t_comb=c.t_comb,
                         t_expert=c.t_expert, slot=ch.slot, objective=ch.objective,
                         makespan=ch.makespan))
    timelines = []
    for frac in (0.0, 0.15, 0.6):
        costs = distsim.derive_costs(64, 128, 32, distsim.HardwareProfile())
        prof = distsim.calibrate_profile(frac, costs, distsim.HardwareProfile())
        for spec in (distsim.StrategySpec("standard_sequential", k=2),
                     distsim.StrategySpec("shared_expert_sequential"),
                     distsim.StrategySpec("scmoe_overlap", pos="pos1"),
                     distsim.StrategySpec("scmoe_overlap", pos="pos2"),
                     distsim.StrategySpec("scmoe_overlap", pos="pos3")):
            nodes = distsim.build_dag(spec, costs, prof)
            tl = distsim.run_sim(nodes)
            kinds = {n.id: n.kind for n in nodes}
            spans = [["comm" if kinds[s.op_id] in distsim.COMM_KINDS else "compute",
                      s.op_id, s.start, s.end] for s in tl.spans]
            timelines.append(dict(frac=frac, label=spec.label,
                                  order=[n.id for n in nodes],
                                  deps={n.id: list(n.deps) for n in nodes},
                                  spans=spans, makespan=tl.makespan,
                                  overlap=distsim.comm_overlap_fraction(nodes, tl)))
    with open(os.path.join(HERE, "sched_cases.json"), "w") as fh:
        json.dump(dict(vectors=vecs, timelines=timelines), fh)


def grad_cases(arch, Rng):
    """Loss and exact gradients of the reference objective (grad.backward,
    grad.py:70-86; LossSpec mean / mse with aux_coeff 0.01) for block pairs
    of every variant, plus the routing they were taken at."""
    sys.path.insert(0, REF_SRC)
    from scmoelab import grad
    out, meta = {}, []
    combos = [dict(variant="scmoe", shortcut_pos="pos2", combine_mode="direct_add", k_routed=1),
              dict(variant="scmoe", shortcut_pos="pos1", combine_mode="cg1", k_routed=1),
              dict(variant="scmoe", shortcut_pos="pos3", combine_mode="cg2", k_routed=1),
              dict(variant="standard", k_routed=2),
              dict(variant="shared", combine_mode="direct_add", k_routed=2)]
    for i, kw in enumerate(combos):
        t, d, h, n, cf = 20, 8, 16, 4, [2.0, 0.75][i % 2]
        cfg = arch.ModelConfig(n_blocks=2, d_model=d, d_hidden=h, n_experts=n,
                               capacity_factor=cf, **kw)
        rng = Rng(300 + i)
        params = arch.init_params(cfg, rng.spawn(0))
        # non-zero biases so their gradients are exercised
        for name, p in arch.named_parameters(params):
            if name.endswith((".b1", ".b2")):
                p += rng.spawn(5).normal(p.shape) * 0.1
        tokens = rng.spawn(1).normal((t, d))
        target = rng.spawn(2).normal((t, d)) if i % 2 else None
        spec = grad.LossSpec(kind="mse", target=target) if target is not None else grad.LossSpec(kind="mean")
        loss, grads, res = grad.backward(cfg, params, tokens, spec)
        p = f"q{i}_"
        out[p + "tokens"] = tokens
        if target is not None:
            out[p + "target"] = target
        out[p + "loss"] = np.asarray(loss)
        out[p + "idx"] = res.trace.moe[0].decision.indices.astype(np.int64)
        out[p + "drop"] = res.trace.moe[0].decision.dropped
        for name, arr in arch.named_parameters(params):
            out[p + "P:" + name] = arr
            out[p + "G:" + name] = grads[name]
        meta.append(dict(t=t, d=d, h=h, n=n, cf=cf, seed=300 + i, mse=target is not None, **kw))
    np.savez_compressed(os.path.join(HERE, "grad_cases.npz"), **out)
    with open(os.path.join(HERE, "grad_cases.json"), "w") as fh:
        json.dump(meta, fh, indent=0)


def model_cases(arch, Rng):
    """Whole-model forwards (arch.forward, arch.py:553-675): stacks of pairs
    with first_layer_pos1, every-block placement (pos1, every variant)."""
    out, meta = {}, []
    combos = [dict(n_blocks=4, variant="scmoe", shortcut_pos="pos2", first_layer_pos1=True),
              dict(n_blocks=4, variant="scmoe", shortcut_pos="pos3", combine_mode="cg1"),
              dict(n_blocks=3, variant="scmoe", shortcut_pos="pos1", moe_frequency="every-block"),
              dict(n_blocks=2, variant="standard", k_routed=2, moe_frequency="every-block"),
              dict(n_blocks=3, variant="shared", moe_frequency="every-block", combine_mode="cg2",
                   pre_layernorm=True)]
    for i, kw in enumerate(combos):
        t, d, h, n = 24, 8, 16, 4
        cfg = arch.ModelConfig(d_model=d, d_hidden=h, n_experts=n, capacity_factor=1.0, **kw)
        rng = Rng(500 + i)
        params = arch.init_params(cfg, rng.spawn(0))
        tokens = rng.spawn(1).normal((t, d))
        o, trace = arch.forward(cfg, params, tokens)
        p = f"m{i}_"
        out[p + "tokens"] = tokens
        out[p + "out"] = o
        for j, m in enumerate(trace.moe):
            out[p + f"idx{j}"] = m.decision.indices.astype(np.int64)
            out[p + f"drop{j}"] = m.decision.dropped
            out[p + f"aux{j}"] = np.asarray(m.aux_loss)
        meta.append(dict(t=t, d=d, h=h, n=n, cf=1.0, seed=500 + i, n_moe=len(trace.moe), **kw))
    np.savez_compressed(os.path.join(HERE, "model_cases.npz"), **out)
    with open(os.path.join(HERE, "model_cases.json"), "w") as fh:
        json.dump(meta, fh, indent=0)


def main():
    arch, distsim, gating, sched, Rng = _import_reference()
    model_cases(arch, Rng)
    gating_cases(gating, Rng)
    layer_and_pair_cases(arch, Rng)
    cfg1_case(arch, Rng)
    sched_cases(sched, distsim)
    grad_cases(arch, Rng)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
