"""CPU oracle for the ScMoE hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in float64 numpy, the reference algorithm of
arXiv 2404.05019's `scmoelab` package for the functions on the ScMoE layer
hot path.  It is the *checker*: only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import it.  The
product (`paper_2404_05019_b200`) never imports or calls this file and has no
CPU fallback.

Parity is PINNED: `tests/test_oracle_golden.py` checks every function below
against golden vectors produced by the real reference
(`tests/golden/make_golden.py` imports `/root/reference/pkg/src/scmoelab`
in the dev container and commits the vectors under `tests/golden/`), plus the
reference's own known-answer tests (`pkg/tests/test_gating.py:49-105`,
`pkg/tests/test_sched.py:27-67`).

Citations are `scmoelab/<file>.py:<line>` relative to
`/root/reference/pkg/src/`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np
from scipy.special import erf

NEG_INF = float("-inf")
_RSQRT2 = 1.0 / math.sqrt(2.0)


# ---------------------------------------------------------------------------
# seeded randomness (scmoelab/numkit.py:26-48): PCG64, sub-streams via
# SeedSequence(seed).spawn(i + 1)[i]


class Rng:
    def __init__(self, seed: int, _gen=None):
        self.seed = int(seed)
        self._gen = _gen if _gen is not None else np.random.Generator(np.random.PCG64(self.seed))

    def spawn(self, index: int) -> "Rng":
        child_seq = np.random.SeedSequence(self.seed).spawn(index + 1)[index]
        return Rng(self.seed, np.random.Generator(np.random.PCG64(child_seq)))

    def normal(self, shape):
        return self._gen.standard_normal(shape)

    def uniform(self, low, high, shape):
        return self._gen.uniform(low, high, shape)

    def integers(self, low, high, shape=None):
        return self._gen.integers(low, high, size=shape)


# ---------------------------------------------------------------------------
# dense numerics (scmoelab/numkit.py:65-105)


def row_softmax(a: np.ndarray) -> np.ndarray:
    """Row softmax with -inf entries mapped to exactly 0 (numkit.py:65-77)."""
    a = np.asarray(a, dtype=np.float64)
    live = a != NEG_INF
    if not live.any(axis=1).all():
        raise ValueError("row_softmax: row with no finite entry")
    row_max = np.max(np.where(live, a, NEG_INF), axis=1, keepdims=True)
    ex = np.where(live, np.exp(np.where(live, a - row_max, 0.0)), 0.0)
    return ex / ex.sum(axis=1, keepdims=True)


def softplus(a):
    """ln(1+e^x) with the linear branch above 30 (numkit.py:80-83)."""
    a = np.asarray(a, dtype=np.float64)
    return np.where(a > 30.0, a, np.log1p(np.exp(np.minimum(a, 30.0))))


def sigmoid(a):
    """Branch-stable logistic (numkit.py:86-93)."""
    a = np.asarray(a, dtype=np.float64)
    e = np.exp(-np.abs(a))
    return np.where(a >= 0, 1.0 / (1.0 + e), e / (1.0 + e))


def gelu(a):
    """Exact erf GELU (numkit.py:96-99)."""
    a = np.asarray(a, dtype=np.float64)
    return 0.5 * a * (1.0 + erf(a * _RSQRT2))


# ---------------------------------------------------------------------------
# parameter containers (scmoelab/arch.py:95-132, gating.py:20-48)


@dataclass
class Expert:
    w1: np.ndarray  # (d, h)
    b1: np.ndarray  # (1, h)
    w2: np.ndarray  # (h, d)
    b2: np.ndarray  # (1, d)


@dataclass
class Gate:
    w_gate: np.ndarray  # (d, N)
    w_noise: np.ndarray  # (d, N)
    k: int
    noise_enabled: bool = False


@dataclass
class Layer:
    experts: List[Expert]
    gate: Gate
    combine_mode: str = "direct_add"
    w_cg: Optional[np.ndarray] = None  # (1, d) cg1 / (2, d) cg2
    shared: Optional[Expert] = None


@dataclass
class Decision:
    logits: np.ndarray
    indices: np.ndarray   # (T, k) int64
    weights: np.ndarray   # (T, k)
    dropped: np.ndarray   # (T, k) bool
    eps: Optional[np.ndarray] = None

    @property
    def k(self):
        return self.indices.shape[1]

    def support_mask(self):
        t, n = self.logits.shape
        m = np.zeros((t, n), dtype=bool)
        m[np.arange(t)[:, None], self.indices] = True
        return m

    def keep_mask(self):
        t, n = self.logits.shape
        m = np.zeros((t, n))
        m[np.arange(t)[:, None], self.indices] = (~self.dropped).astype(np.float64)
        return m


# ---------------------------------------------------------------------------
# gating (scmoelab/gating.py:93-170)


def gate_logits(x, gate: Gate, eps=None, rng: Optional[Rng] = None):
    """H = x W_gate (+ eps * softplus(x W_noise)) (gating.py:93-107)."""
    x = np.asarray(x, dtype=np.float64)
    clean = x @ gate.w_gate
    if not gate.noise_enabled:
        return clean, None
    if eps is None:
        if rng is None:
            raise ValueError("noise enabled but no rng and no recorded draws")
        eps = rng.normal(clean.shape)
    return clean + eps * softplus(x @ gate.w_noise), eps


def topk_indices(h, k: int) -> np.ndarray:
    """k largest per row, rank order by value, ties to lowest index
    (gating.py:110-116: stable argsort of -h)."""
    h = np.asarray(h, dtype=np.float64)
    if k > h.shape[1]:
        raise ValueError(f"k={k} > N={h.shape[1]}")
    return np.argsort(-h, axis=1, kind="stable")[:, :k]


def _masked_weights(h, idx):
    """Softmax over the selected logits only (gating.py:125-129)."""
    t = h.shape[0]
    rows = np.arange(t)[:, None]
    masked = np.full_like(h, NEG_INF)
    masked[rows, idx] = h[rows, idx]
    return row_softmax(masked)[rows, idx]


def select_topk(h, k: int, eps=None) -> Decision:
    h = np.asarray(h, dtype=np.float64)
    idx = topk_indices(h, k)
    return Decision(logits=h, indices=idx, weights=_masked_weights(h, idx),
                    dropped=np.zeros(idx.shape, dtype=bool), eps=eps)


def expert_quota(capacity_factor: float, n_tokens: int, k: int, n_experts: int) -> int:
    """ceil(cf*T*k/N) evaluated left to right in float64 (gating.py:134-135)."""
    return int(math.ceil(capacity_factor * n_tokens * k / n_experts))


def capacity_slots(indices: np.ndarray, n_experts: int) -> np.ndarray:
    """Derived oracle: slot of selection (t, j) = number of
    earlier selections of the same expert in token-major order.  This is the
    count `apply_capacity` (gating.py:146-154) compares with the quota."""
    flat = np.asarray(indices, dtype=np.int64).reshape(-1)
    onehot = (flat[:, None] == np.arange(n_experts)[None, :]).astype(np.int64)
    before = np.cumsum(onehot, axis=0) - onehot
    return before[np.arange(flat.size), flat].reshape(np.asarray(indices).shape)


def apply_capacity(dec: Decision, capacity_factor: float, n_experts: int,
                   n_tokens: int) -> Decision:
    """Drop selections past the quota, token-major (t, then rank) order;
    weights untouched (gating.py:138-156).  Note the counter only advances
    on *kept* selections, so slot >= quota <=> dropped."""
    quota = expert_quota(capacity_factor, n_tokens, dec.k, n_experts)
    used = np.zeros(n_experts, dtype=np.int64)
    dropped = dec.dropped.copy()
    for t in range(dec.indices.shape[0]):
        for j in range(dec.k):
            e = dec.indices[t, j]
            if used[e] >= quota:
                dropped[t, j] = True
            else:
                used[e] += 1
    return Decision(dec.logits, dec.indices, dec.weights, dropped, dec.eps)


def load_balance_loss(dec: Decision, n_experts: int) -> float:
    """N * sum_i f_i P_i with pre-drop f (gating.py:159-170, arch.py:436-439)."""
    t = dec.logits.shape[0]
    f = np.bincount(dec.indices.ravel(), minlength=n_experts) / float(t * dec.k)
    p = row_softmax(dec.logits).mean(axis=0)
    return float(n_experts * (f * p).sum())


def decision_from_indices(h, indices, dropped, eps=None) -> Decision:
    """Replay pinned routing (arch.py:395-402)."""
    h = np.asarray(h, dtype=np.float64)
    indices = np.asarray(indices, dtype=np.int64)
    return Decision(h, indices.copy(), _masked_weights(h, indices),
                    np.asarray(dropped, dtype=bool).copy(), eps)


def standard_routing(h, k, capacity_factor) -> Decision:
    """select_topk then apply_capacity (arch.py:442-444)."""
    h = np.asarray(h, dtype=np.float64)
    return apply_capacity(select_topk(h, k), capacity_factor, h.shape[1], h.shape[0])


# ---------------------------------------------------------------------------
# layer (scmoelab/arch.py:349-504)


def expert_forward(x, e: Expert):
    """gelu(x W1 + b1) W2 + b2 (arch.py:349-351)."""
    return gelu(np.asarray(x, dtype=np.float64) @ e.w1 + e.b1) @ e.w2 + e.b2


def combine(se_out, routed_out, x, mode: str, w_cg=None):
    """direct_add / CG-1 sigmoid / CG-2 2-way softmax on x_cur (arch.py:380-392)."""
    if mode == "direct_add":
        return se_out + routed_out
    logits = np.asarray(x, dtype=np.float64) @ np.asarray(w_cg).T
    if mode == "cg1":
        return sigmoid(logits) * se_out + routed_out
    coef = row_softmax(logits)
    return coef[:, :1] * se_out + coef[:, 1:2] * routed_out


def routed_sum_dense(x_src, experts: Sequence[Expert], weight_matrix):
    """sum_i w[:, i] * E_i(x_src) with every used expert evaluated on ALL
    rows — the reference's dense algorithm (arch.py:418-433)."""
    out = None
    for i, e in enumerate(experts):
        col = weight_matrix[:, i:i + 1]
        if not col.any():
            continue
        term = col * expert_forward(x_src, e)
        out = term if out is None else out + term
    return np.zeros_like(np.asarray(x_src, dtype=np.float64)) if out is None else out


def routed_moe(x_src, layer: Layer, k: int, capacity_factor: float, eps=None,
               rng=None, pinned_indices=None, pinned_dropped=None):
    """(out, decision, aux) of the routed mixture (arch.py:463-486)."""
    h, eps_used = gate_logits(x_src, layer.gate, eps=eps, rng=rng)
    if pinned_indices is not None:
        if pinned_dropped is None:
            pinned_dropped = np.zeros(np.shape(pinned_indices), dtype=bool)
        dec = decision_from_indices(h, pinned_indices, pinned_dropped, eps_used)
    else:
        dec = standard_routing(h, k, capacity_factor)
        dec.eps = eps_used
    support = dec.support_mask()
    probs = row_softmax(np.where(support, h, NEG_INF))
    weights_used = probs * dec.keep_mask()
    out = routed_sum_dense(x_src, layer.experts, weights_used)
    aux = load_balance_loss(dec, h.shape[1])
    return out, dec, aux


def moe_standard(x, layer: Layer, capacity_factor: float, k: int, eps=None, rng=None,
                 pinned_indices=None, pinned_dropped=None):
    """Top-k MoE without shared expert (arch.py:489-493)."""
    return routed_moe(x, layer, k, capacity_factor, eps=eps, rng=rng,
                      pinned_indices=pinned_indices, pinned_dropped=pinned_dropped)


def moe_shared(x, layer: Layer, capacity_factor: float, k: int, routed_src=None,
               eps=None, rng=None, pinned_indices=None, pinned_dropped=None):
    """ScMoE / shared-expert layer: combine(SE(x), routed(src), x)
    (arch.py:496-504)."""
    src = x if routed_src is None else routed_src
    routed, dec, aux = routed_moe(src, layer, k, capacity_factor, eps=eps, rng=rng,
                                  pinned_indices=pinned_indices,
                                  pinned_dropped=pinned_dropped)
    se = expert_forward(x, layer.shared)
    return combine(se, routed, x, layer.combine_mode, layer.w_cg), dec, aux


# ---------------------------------------------------------------------------
# block-pair wiring (scmoelab/arch.py:354-377, 540-631)


@dataclass
class Attention:
    w_q: np.ndarray
    w_k: np.ndarray
    w_v: np.ndarray
    w_o: np.ndarray


def attention_forward(x, a: Attention, d_model: int):
    """Single-head unmasked SDPA, 1/sqrt(d_model) scale (arch.py:354-358)."""
    q, k, v = x @ a.w_q, x @ a.w_k, x @ a.w_v
    return row_softmax((q @ k.T) * (1.0 / np.sqrt(d_model))) @ v @ a.w_o


def layer_norm(x):
    """Parameter-free row LN, eps 1e-6 (arch.py:361-377)."""
    mu = x.mean(axis=1, keepdims=True)
    return (x - mu) / np.sqrt(x.var(axis=1, keepdims=True) + 1e-6)


@dataclass
class PairParams:
    attn_prev: Attention
    mlp_prev: Expert
    attn_cur: Attention
    moe: Layer


def init_pair(d: int, h: int, n_experts: int, rng: Rng, variant: str = "scmoe",
              k: int = 1, combine_mode: str = "direct_add",
              noise_enabled: bool = False) -> PairParams:
    """Draw order of init_params for one block pair (arch.py:158-190):
    attn(prev) 4x(d,d), MLP W1,W2, attn(cur) 4x(d,d), N experts (W1,W2 each),
    shared (W1,W2) if any, W_gate, W_noise, W_cg if CG.  Scale 1/sqrt(d),
    zero biases."""
    s = 1.0 / np.sqrt(d)

    def expert():
        w1 = rng.normal((d, h)) * s
        w2 = rng.normal((h, d)) * s
        return Expert(w1, np.zeros((1, h)), w2, np.zeros((1, d)))

    def attn():
        return Attention(*(rng.normal((d, d)) * s for _ in range(4)))

    a_prev = attn()
    mlp = expert()
    a_cur = attn()
    experts = [expert() for _ in range(n_experts)]
    shared = expert() if variant in ("shared", "scmoe") else None
    wg = rng.normal((d, n_experts)) * s
    wn = rng.normal((d, n_experts)) * s
    w_cg = None
    if combine_mode != "direct_add":
        w_cg = rng.normal((1 if combine_mode == "cg1" else 2, d)) * s
    layer = Layer(experts, Gate(wg, wn, k, noise_enabled), combine_mode, w_cg, shared)
    return PairParams(a_prev, mlp, a_cur, layer)


def block_pair_forward(p: PairParams, h_in, variant: str, pos: Optional[str],
                       capacity_factor: float, k: int, pre_layernorm: bool = False,
                       eps=None, rng=None, pinned_indices=None, pinned_dropped=None):
    """Block-MLP + Block-MoE pair (arch.py:580-631); returns (out, decision,
    aux, taps) with taps = dict of the intermediate representations."""
    d = h_in.shape[1]
    feed = layer_norm if pre_layernorm else (lambda z: z)
    h_mh_prev = h_in + attention_forward(feed(h_in), p.attn_prev, d)
    h_mlp_prev = h_mh_prev + expert_forward(feed(h_mh_prev), p.mlp_prev)
    h_mh_cur = h_mlp_prev + attention_forward(feed(h_mlp_prev), p.attn_cur, d)
    x_cur = feed(h_mh_cur)
    kw = dict(eps=eps, rng=rng, pinned_indices=pinned_indices,
              pinned_dropped=pinned_dropped)
    if variant == "scmoe":
        src = {"pos1": h_mlp_prev, "pos2": h_mh_prev, "pos3": h_in}[pos]
        f, dec, aux = moe_shared(x_cur, p.moe, capacity_factor, k, routed_src=src, **kw)
    elif variant == "shared":
        src = x_cur
        f, dec, aux = moe_shared(x_cur, p.moe, capacity_factor, k, **kw)
    else:
        src = x_cur
        f, dec, aux = moe_standard(x_cur, p.moe, capacity_factor, k, **kw)
    taps = dict(h_mh_prev=h_mh_prev, h_mlp_prev=h_mlp_prev, h_mh_cur=h_mh_cur,
                x_cur=x_cur, src=src)
    return h_mh_cur + f, dec, aux, taps


# ---------------------------------------------------------------------------
# scheduler and overlap metric (scmoelab/sched.py:73-98, distsim.py:456-469)


def choose_slot(comp: Sequence[float], t_disp: float, t_comb: float, t_expert: float):
    """argmin_K |pre(K)-t_disp| + |post(K)-t_comb|, ties to smallest K;
    returns (slot, objective, makespan) (sched.py:73-98)."""
    best = None
    for kk in range(len(comp) + 1):
        pre, post = sum(comp[:kk]), sum(comp[kk:])
        obj = abs(pre - t_disp) + abs(post - t_comb)
        if best is None or obj < best[1]:
            best = (kk, obj, max(pre, t_disp) + t_expert + max(post, t_comb))
    return best


def comm_overlap_fraction(spans: Sequence[Tuple[str, float, float]]) -> float:
    """spans = (kind, start, end) with kind in {"comm", "compute"}; the comm
    time covered by the union of compute spans over total comm time, 1.0
    without comm (distsim.py:446-469)."""
    comp = sorted((a, b) for kind, a, b in spans if kind != "comm")
    merged: List[List[float]] = []
    for a, b in comp:
        if merged and a <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], b)
        else:
            merged.append([a, b])
    total = hidden = 0.0
    for kind, a, b in spans:
        if kind != "comm":
            continue
        total += b - a
        for ca, cb in merged:
            hidden += max(0.0, min(cb, b) - max(ca, a))
    return 1.0 if total == 0.0 else hidden / total


def allclose_scaled(a, b, rtol: float) -> Tuple[bool, float]:
    """The parity check used by the tests (SURVEY §7 hard part 2):
    |a-b| <= atol + rtol*|b| with atol = rtol*max|b|.  Returns (ok, worst
    ratio of |a-b| to the bound)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    atol = rtol * float(np.max(np.abs(b))) if b.size else 0.0
    bound = atol + rtol * np.abs(b)
    bound = np.where(bound == 0, 1e-300, bound)
    worst = float(np.max(np.abs(a - b) / bound)) if b.size else 0.0
    return worst <= 1.0, worst


# ---------------------------------------------------------------------------
# whole model (scmoelab/arch.py:167-196 init, 553-665 model_forward)


@dataclass
class BlockP:
    attn: Attention
    feed: object          # Expert (Block-MLP) or Layer (Block-MoE)


def init_model(n_blocks: int, d: int, h: int, n_experts: int, rng: Rng,
               moe_frequency: str = "every-second-block", variant: str = "scmoe", k: int = 1,
               combine_mode: str = "direct_add", noise_enabled: bool = False):
    """init_params draw order for any block count (arch.py:167-196): per block
    attention (4 x (d,d)), then the feed: Block-MLP (W1, W2) or the MoE layer
    (N experts, shared, W_gate, W_noise, W_cg).  MoE blocks are the odd ones
    (every-second-block) or all (every-block), arch.py:193-196."""
    s = 1.0 / np.sqrt(d)

    def expert():
        w1 = rng.normal((d, h)) * s
        w2 = rng.normal((h, d)) * s
        return Expert(w1, np.zeros((1, h)), w2, np.zeros((1, d)))

    blocks = []
    for i in range(n_blocks):
        attn = Attention(*(rng.normal((d, d)) * s for _ in range(4)))
        is_moe = moe_frequency == "every-block" or i % 2 == 1
        if is_moe:
            experts = [expert() for _ in range(n_experts)]
            shared = expert() if variant in ("shared", "scmoe") else None
            wg = rng.normal((d, n_experts)) * s
            wn = rng.normal((d, n_experts)) * s
            w_cg = None
            if combine_mode != "direct_add":
                w_cg = rng.normal((1 if combine_mode == "cg1" else 2, d)) * s
            feed = Layer(experts, Gate(wg, wn, k, noise_enabled), combine_mode, w_cg, shared)
        else:
            feed = expert()
        blocks.append(BlockP(attn, feed))
    return blocks


def model_forward(blocks, tokens, variant: str, pos: Optional[str], capacity_factor: float,
                  k: int, moe_frequency: str = "every-second-block",
                  first_layer_pos1: bool = False, pre_layernorm: bool = False,
                  pinned=None):
    """arch.model_forward (arch.py:553-665) value mode; `pinned` is an optional
    list of (indices, dropped) per MoE layer.  Returns (out, decisions, auxes)."""
    d = tokens.shape[1]
    feed = layer_norm if pre_layernorm else (lambda z: z)
    h = np.asarray(tokens, dtype=np.float64)
    decs, auxes = [], []

    def moe_call(layer, x_cur, src, j):
        kw = {}
        if pinned is not None:
            kw = dict(pinned_indices=pinned[j][0], pinned_dropped=pinned[j][1])
        if variant == "scmoe":
            return moe_shared(x_cur, layer, capacity_factor, k, routed_src=src, **kw)
        if variant == "shared":
            return moe_shared(x_cur, layer, capacity_factor, k, **kw)
        return moe_standard(x_cur, layer, capacity_factor, k, **kw)

    if moe_frequency == "every-second-block":
        for pair in range(len(blocks) // 2):
            prev_b, cur_b = blocks[2 * pair], blocks[2 * pair + 1]
            h_in = h
            h_mh_prev = h_in + attention_forward(feed(h_in), prev_b.attn, d)
            h_mlp_prev = h_mh_prev + expert_forward(feed(h_mh_prev), prev_b.feed)
            h_mh_cur = h_mlp_prev + attention_forward(feed(h_mlp_prev), cur_b.attn, d)
            x_cur = feed(h_mh_cur)
            p = "pos1" if (variant == "scmoe" and first_layer_pos1 and pair == 0) else pos
            src = {"pos1": h_mlp_prev, "pos2": h_mh_prev, "pos3": h_in}.get(p, x_cur) \
                if variant == "scmoe" else x_cur
            f, dec, aux = moe_call(cur_b.feed, x_cur, src, pair)
            decs.append(dec)
            auxes.append(aux)
            h = h_mh_cur + f
    else:
        for i, b in enumerate(blocks):
            h_in = h
            h_mh = h_in + attention_forward(feed(h_in), b.attn, d)
            x_cur = feed(h_mh)
            src = h_in if variant == "scmoe" else x_cur
            f, dec, aux = moe_call(b.feed, x_cur, src, i)
            decs.append(dec)
            auxes.append(aux)
            h = h_mh + f
    return h, decs, auxes


# ---------------------------------------------------------------------------
# DGMoE: dual top-1 gating with the distinct-expert constraint
# (scmoelab/arch.py:447-460 dual_routing, 507-533 moe_dual_gating)


def dual_routing(h_cur, h_prev, constraint: bool, capacity_factor: float):
    """(dec_cur, dec_prev): top-1 on the preceding representation with
    capacity; on the current one the top-1, replaced by the runner-up when it
    equals the preceding pick (constraint on), then capacity."""
    h_cur = np.asarray(h_cur, dtype=np.float64)
    n, t = h_prev.shape[1], h_prev.shape[0]
    dec_prev = apply_capacity(select_topk(h_prev, 1), capacity_factor, n, t)
    top2 = topk_indices(h_cur, 2)
    idx = top2[:, :1].copy()
    if constraint:
        clash = idx[:, 0] == dec_prev.indices[:, 0]
        idx[clash, 0] = top2[clash, 1]
    dec_cur = decision_from_indices(h_cur, idx, np.zeros((t, 1), dtype=bool))
    return apply_capacity(dec_cur, capacity_factor, n, t), dec_prev


def moe_dual_gating(x_cur, x_prev, layer: Layer, capacity_factor: float, constraint: bool,
                    pinned=None, eps=None, eps_prev=None):
    """routed_sum(x_cur, w_cur) + routed_sum(x_prev, w_prev); aux from the
    current gating (arch.py:507-533).  pinned = ((idx_cur, drop_cur),
    (idx_prev, drop_prev)) replays the routing; eps / eps_prev are the noisy
    gate's recorded draws of the two gatings (arch.py:514-515)."""
    h_prev, _ = gate_logits(x_prev, layer.gate, eps=eps_prev)
    h_cur, _ = gate_logits(x_cur, layer.gate, eps=eps)
    if pinned is not None:
        dec_cur = decision_from_indices(h_cur, pinned[0][0], pinned[0][1])
        dec_prev = decision_from_indices(h_prev, pinned[1][0], pinned[1][1])
    else:
        dec_cur, dec_prev = dual_routing(h_cur, h_prev, constraint, capacity_factor)

    def wmat(h, dec):
        return row_softmax(np.where(dec.support_mask(), h, NEG_INF)) * dec.keep_mask()

    out = routed_sum_dense(x_cur, layer.experts, wmat(h_cur, dec_cur)) + \
        routed_sum_dense(x_prev, layer.experts, wmat(h_prev, dec_prev))
    return out, dec_cur, dec_prev, load_balance_loss(dec_cur, h_cur.shape[1])


def dgmoe_pair_forward(p: PairParams, h_in, capacity_factor: float, constraint: bool = True,
                       pre_layernorm: bool = False, pinned=None):
    """Block pair with the DGMoE feed; the preceding gating reads h_mh_prev
    (arch.py:606-609).  Returns (out, dec_cur, dec_prev, aux)."""
    d = h_in.shape[1]
    feed = layer_norm if pre_layernorm else (lambda z: z)
    h_mh_prev = h_in + attention_forward(feed(h_in), p.attn_prev, d)
    h_mlp_prev = h_mh_prev + expert_forward(feed(h_mh_prev), p.mlp_prev)
    h_mh_cur = h_mlp_prev + attention_forward(feed(h_mlp_prev), p.attn_cur, d)
    x_cur = feed(h_mh_cur)
    f, dc, dp, aux = moe_dual_gating(x_cur, h_mh_prev, p.moe, capacity_factor, constraint, pinned)
    return h_mh_cur + f, dc, dp, aux
