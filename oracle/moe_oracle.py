"""CPU restatement of the reference MoE-layer hot path (TEST INFRASTRUCTURE ONLY).

This module is the parity checker for the B200 path.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference`` legs
of ``bench.py`` may import it.  The product package never does: it fails
loudly when its CUDA extension is missing instead of falling back here.

Everything is numpy float64, mirroring the reference simulator ``moefold``
(``/root/reference/pkg/src/moefold``).  Each function names the reference
lines whose behaviour it restates.  The restatement is *pinned*: the golden
vectors under ``tests/golden/`` were produced by importing the reference
itself (``tests/golden/make_golden.py``) and ``tests/test_oracle_golden.py``
checks this module against them (integers bit-exact, floats to 1e-12).

Two pieces have no reference implementation and are builder-defined (parity
for them is pinned only by this restatement plus finite-difference checks):
the SwiGLU expert (``act="swiglu"``) and the dense shared expert.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

GELU_C = math.sqrt(2.0 / math.pi)


# ----------------------------------------------------------------------------
# router (reference: pkg/src/moefold/router.py)
# ----------------------------------------------------------------------------

def softmax_rows(z: np.ndarray) -> np.ndarray:
    """Max-shifted row softmax -- router.py:112-117."""
    z = np.asarray(z, dtype=np.float64)
    m = z.max(axis=1, keepdims=True)
    ex = np.exp(z - m)
    return ex / ex.sum(axis=1, keepdims=True)


def sigmoid(z: np.ndarray) -> np.ndarray:
    """router.py:149."""
    return 1.0 / (1.0 + np.exp(-np.asarray(z, dtype=np.float64)))


def select_topk(scores: np.ndarray, k: int) -> np.ndarray:
    """Best-first top-k, ties to the lower expert id -- router.py:120-124."""
    return np.argsort(-scores, axis=1, kind="stable")[:, :k]


@dataclass
class Routing:
    experts: np.ndarray  # [n, k] int64, best first
    gates: np.ndarray  # [n, k] float64
    kept: np.ndarray  # [n, k] bool
    scores: np.ndarray  # [n, E] float64


def route_logits(logits: np.ndarray, k: int, gate_fn: str = "softmax",
                 renormalize: bool = False) -> Routing:
    """Scores, top-k and gates from router logits -- router.py:145-162.

    The reference forms logits as ``x @ w_g``; feeding logits directly is the
    same as calling ``compute_gates(logits, w_g=eye(E))``.
    """
    logits = np.asarray(logits, dtype=np.float64)
    scores = softmax_rows(logits) if gate_fn == "softmax" else sigmoid(logits)
    experts = select_topk(scores, k)
    gates = np.take_along_axis(scores, experts, axis=1)
    if renormalize:
        gates = gates / gates.sum(axis=1, keepdims=True)
    kept = np.ones(experts.shape, dtype=bool)
    return Routing(experts.astype(np.int64), gates, kept, scores)


def capacity_limit(capacity_factor: float, l_scope: int, num_experts: int) -> int:
    """floor(CF * L / E), at least one -- router.py:165-168 (no k factor)."""
    return max(1, math.floor(capacity_factor * l_scope / num_experts))


def apply_capacity(experts: np.ndarray, gates: np.ndarray, kept: np.ndarray,
                   positions: np.ndarray, cap: int, num_experts: int,
                   priority: str = "position") -> np.ndarray:
    """Admit pairs per expert up to ``cap`` in priority order -- router.py:171-206.

    Position priority walks (position, slot); probability priority walks
    (-gate, position, slot).  Returns the new kept mask.
    """
    n, k = experts.shape
    flat_e = experts.reshape(-1)
    out = kept.copy().reshape(-1)
    pos = np.repeat(np.asarray(positions, dtype=np.int64), k)
    slot = np.tile(np.arange(k), n)
    if priority == "position":
        order = np.lexsort((slot, pos))
    else:
        order = np.lexsort((slot, pos, -gates.reshape(-1)))
    used = np.zeros(num_experts, dtype=np.int64)
    for idx in order:
        if not out[idx]:
            continue
        e = flat_e[idx]
        if used[e] < cap:
            used[e] += 1
        else:
            out[idx] = False
    return out.reshape(n, k)


def capacity_rank_vectorized(experts: np.ndarray, cap: int, num_experts: int) -> np.ndarray:
    """Closed form of position-priority capacity for rows already in position
    order: pair (t, s) survives iff fewer than ``cap`` earlier tokens chose the
    same expert (a token's k experts are distinct).  Equivalent to
    ``apply_capacity(..., priority="position")``."""
    n, k = experts.shape
    flat = experts.reshape(-1)
    onehot = np.zeros((flat.size, num_experts), dtype=np.int64)
    onehot[np.arange(flat.size), flat] = 1
    rank = np.cumsum(onehot, axis=0) - onehot
    return (rank[np.arange(flat.size), flat] < cap).reshape(n, k)


def load_stats(experts: np.ndarray, kept: np.ndarray, scores: Optional[np.ndarray],
               num_experts: int):
    """Kept pairs per expert, max/mean imbalance, Switch aux loss -- router.py:279-301."""
    counts = np.bincount(experts.reshape(-1)[kept.reshape(-1)], minlength=num_experts)
    mean = counts.sum() / num_experts
    imbalance = float(counts.max() / mean) if mean > 0 else float("nan")
    if scores is None or experts.shape[0] == 0:
        aux = float("nan")
    else:
        f = np.bincount(experts[:, 0], minlength=num_experts) / experts.shape[0]
        p = (scores / scores.sum(axis=1, keepdims=True)).mean(axis=0)
        aux = float(num_experts * np.dot(f, p))
    return counts.astype(np.int64), imbalance, aux


def full_sequence_kept(experts_list: Sequence[np.ndarray], gates_list: Sequence[np.ndarray],
                       positions_list: Sequence[np.ndarray], seq_len: int,
                       capacity_factor: float, num_experts: int,
                       priority: str = "position") -> List[np.ndarray]:
    """Full-sequence dropping over the shards of a sequence group --
    router.py:209-269: union the pairs of every shard, apply capacity per
    sequence of ``seq_len`` tokens, and map the flags back per shard."""
    pos = np.concatenate([np.asarray(p, dtype=np.int64) for p in positions_list])
    ex = np.concatenate(list(experts_list))
    gt = np.concatenate(list(gates_list))
    order = np.argsort(pos, kind="stable")
    pos_s, ex_s, gt_s = pos[order], ex[order], gt[order]
    kept_s = np.ones(ex_s.shape, dtype=bool)
    seq = pos_s // seq_len
    cap = capacity_limit(capacity_factor, seq_len, num_experts)
    for sid in np.unique(seq):
        m = seq == sid
        kept_s[m] = apply_capacity(ex_s[m], gt_s[m], kept_s[m], pos_s[m], cap,
                                   num_experts, priority)
    lookup = {int(p): i for i, p in enumerate(pos_s)}
    out = []
    for p in positions_list:
        out.append(np.stack([kept_s[lookup[int(q)]] for q in p]) if len(p)
                   else np.zeros((0, ex.shape[1]), dtype=bool))
    return out


# ----------------------------------------------------------------------------
# dispatch plan, permute, combine (reference: pkg/src/moefold/dispatcher.py)
# ----------------------------------------------------------------------------

@dataclass
class Plan:
    permutation: np.ndarray  # [P] flat token*k+slot, send order
    send_counts: np.ndarray  # [ep, local]
    gates: np.ndarray  # [P]
    n_tokens: int
    k: int

    @property
    def pair_tokens(self):
        return self.permutation // self.k

    @property
    def pair_slots(self):
        return self.permutation % self.k


def build_dispatch_plan(experts: np.ndarray, gates: np.ndarray, kept: np.ndarray,
                        ep_size: int, local_experts: int) -> Plan:
    """Kept pairs ordered by (dest rank, local expert, token, slot), i.e. a
    stable counting sort by global expert id -- dispatcher.py:96-131."""
    n, k = experts.shape
    idx = np.flatnonzero(kept.reshape(-1))
    e = experts.reshape(-1)[idx]
    # one stable sort on the global expert id == lexsort((slot, token, le, dest))
    order = np.argsort(e, kind="stable")
    perm = idx[order]
    counts = np.bincount(e, minlength=ep_size * local_experts).reshape(ep_size, local_experts)
    return Plan(perm, counts.astype(np.int64), gates.reshape(-1)[perm], n, k)


def permute(x: np.ndarray, plan: Plan) -> np.ndarray:
    """Row gather into send order -- dispatcher.py:134-142."""
    return np.asarray(x, dtype=np.float64)[plan.pair_tokens]


def unpermute_combine(rows: np.ndarray, plan: Plan, hidden: int) -> np.ndarray:
    """Gate-weighted scatter-add back to token order -- dispatcher.py:145-157."""
    out = np.zeros((plan.n_tokens, hidden))
    np.add.at(out, plan.pair_tokens, plan.gates[:, None] * np.asarray(rows, dtype=np.float64))
    return out


# ----------------------------------------------------------------------------
# experts (reference: pkg/src/moefold/experts.py; SwiGLU is builder-defined)
# ----------------------------------------------------------------------------

def act_fwd(pre: np.ndarray, act: str) -> np.ndarray:
    """experts.py:23-28 (relu, tanh-gelu)."""
    if act == "relu":
        return np.maximum(pre, 0.0)
    inner = GELU_C * (pre + 0.044715 * pre ** 3)
    return 0.5 * pre * (1.0 + np.tanh(inner))


def act_grad(pre: np.ndarray, act: str) -> np.ndarray:
    """experts.py:31-37."""
    if act == "relu":
        return (pre > 0.0).astype(np.float64)
    inner = GELU_C * (pre + 0.044715 * pre ** 3)
    t = np.tanh(inner)
    return 0.5 * (1.0 + t) + 0.5 * pre * (1.0 - t * t) * GELU_C * (1.0 + 3 * 0.044715 * pre ** 2)


def silu(z):
    return z / (1.0 + np.exp(-z))


def silu_grad(z):
    s = 1.0 / (1.0 + np.exp(-z))
    return s * (1.0 + z * (1.0 - s))


@dataclass
class Expert:
    """One expert (or one ETP shard of it).

    MLP (reference): ``w1`` [H, F], ``w2`` [F, H], ``act`` relu|gelu.
    SwiGLU (builder-defined): ``w1`` is [H, 2F] = [gate | up], ``w2`` [F, H],
    y = (silu(x Wg) * (x Wu)) W2.  ETP shards slice gate and up column-wise
    and W2 row-wise, so partials sum to the unsharded output.
    """
    w1: np.ndarray
    w2: np.ndarray
    act: str = "relu"


def expert_forward(x: np.ndarray, ex: Expert) -> Tuple[np.ndarray, np.ndarray]:
    """experts.py:130-143; returns (out, pre)."""
    x = np.asarray(x, dtype=np.float64)
    pre = x @ ex.w1
    if ex.act == "swiglu":
        f = pre.shape[1] // 2
        h = silu(pre[:, :f]) * pre[:, f:]
    else:
        h = act_fwd(pre, ex.act)
    return h @ ex.w2, pre


def expert_backward(dy: np.ndarray, x: np.ndarray, pre: np.ndarray, ex: Expert,
                    relu_mask: Optional[np.ndarray] = None):
    """experts.py:146-172: recompute the activation from ``pre``; returns
    (dx_partial, dw1, dw2).  ``relu_mask`` optionally supplies relu'(pre) as
    observed by the implementation under test: where a pre-activation lies
    within rounding of 0 the two sides may legitimately disagree on the sign
    (the discontinuity oracle.py:176-186 skips as an unstable probe)."""
    dy = np.asarray(dy, dtype=np.float64)
    if ex.act == "swiglu":
        f = pre.shape[1] // 2
        g, u = pre[:, :f], pre[:, f:]
        h = silu(g) * u
        dh = dy @ ex.w2.T
        dpre = np.concatenate([dh * u * silu_grad(g), dh * silu(g)], axis=1)
    else:
        h = act_fwd(pre, ex.act)
        if ex.act == "relu" and relu_mask is not None:
            h = np.where(relu_mask, pre, 0.0)
        dh = dy @ ex.w2.T
        grad = act_grad(pre, ex.act) if relu_mask is None or ex.act != "relu" else relu_mask.astype(np.float64)
        dpre = dh * grad
    dw2 = h.T @ dy
    dw1 = x.T @ dpre
    return dpre @ ex.w1.T, dw1, dw2


# ----------------------------------------------------------------------------
# one rank's MoE layer, forward + backward (dispatcher.py:246-510)
# ----------------------------------------------------------------------------

@dataclass
class LayerConfig:
    k: int
    gate_fn: str = "softmax"
    renormalize: bool = False
    capacity_factor: Optional[float] = None
    drop_priority: str = "position"


@dataclass
class LayerState:
    x: np.ndarray
    routing: Routing
    plan: Plan
    pres: Dict[int, np.ndarray] = field(default_factory=dict)
    xs: Dict[int, np.ndarray] = field(default_factory=dict)
    y_perm: Optional[np.ndarray] = None
    logits: Optional[np.ndarray] = None


def layer_forward(x: np.ndarray, logits: np.ndarray, experts: Sequence[Expert],
                  cfg: LayerConfig, positions: Optional[np.ndarray] = None,
                  kept_override: Optional[np.ndarray] = None,
                  shared: Optional[Expert] = None) -> Tuple[np.ndarray, LayerState]:
    """Forward of one rank's token block against the full expert set.

    Expert outputs do not depend on the EP/ETP factorisation (each pair row is
    independent and ETP partials sum exactly), so one rank's output equals the
    reference ``moe_forward`` output for that rank given the same routing
    scope.  Sub-sequence capacity scope = the rank's rows
    (dispatcher.py:299-306); ``kept_override`` injects full-sequence flags.
    ``shared`` adds a dense expert applied to every token (builder-defined).
    """
    x = np.asarray(x, dtype=np.float64)
    n, hidden = x.shape
    E = len(experts)
    r = route_logits(logits, cfg.k, cfg.gate_fn, cfg.renormalize)
    if positions is None:
        positions = np.arange(n, dtype=np.int64)
    if kept_override is not None:
        r.kept = np.asarray(kept_override, dtype=bool).copy()
    elif cfg.capacity_factor is not None:
        cap = capacity_limit(cfg.capacity_factor, n, E)
        r.kept = apply_capacity(r.experts, r.gates, r.kept, positions, cap, E, cfg.drop_priority)
    plan = build_dispatch_plan(r.experts, r.gates, r.kept, 1, E)
    sent = permute(x, plan)
    e_sorted = r.experts.reshape(-1)[plan.permutation]
    y_perm = np.zeros_like(sent)
    st = LayerState(x, r, plan, logits=np.asarray(logits, dtype=np.float64))
    for e in range(E):
        rows = np.flatnonzero(e_sorted == e)
        if rows.size:
            out, pre = expert_forward(sent[rows], experts[e])
            y_perm[rows] = out
            st.pres[e] = pre
            st.xs[e] = sent[rows]
    st.y_perm = y_perm
    out = unpermute_combine(y_perm, plan, hidden)
    if shared is not None:
        sy, spre = expert_forward(x, shared)
        out = out + sy
        st.pres[-1] = spre
    return out, st


def layer_backward(u: np.ndarray, st: LayerState, experts: Sequence[Expert], cfg: LayerConfig,
                   w_g: Optional[np.ndarray] = None, shared: Optional[Expert] = None,
                   relu_masks: Optional[Dict[int, np.ndarray]] = None):
    """Backward of ``sum(u * forward)`` -- dispatcher.py:409-500.

    Returns (dx, dlogits, dwg or None, dw1 list, dw2 list, shared grads or None).
    ``dx`` includes the router term ``dz @ w_g.T`` when ``w_g`` is given
    (dispatcher.py:489-490).
    """
    u = np.asarray(u, dtype=np.float64)
    plan, r = st.plan, st.routing
    n, hidden = st.x.shape
    E = len(experts)
    pt = plan.pair_tokens
    dy_perm = plan.gates[:, None] * u[pt]
    dgate_pairs = (u[pt] * st.y_perm).sum(axis=1)
    e_sorted = r.experts.reshape(-1)[plan.permutation]
    dx_perm = np.zeros_like(dy_perm)
    dw1 = [np.zeros_like(ex.w1) for ex in experts]
    dw2 = [np.zeros_like(ex.w2) for ex in experts]
    for e in range(E):
        rows = np.flatnonzero(e_sorted == e)
        if rows.size:
            mask = None if relu_masks is None else relu_masks.get(e)
            d, g1, g2 = expert_backward(dy_perm[rows], st.xs[e], st.pres[e], experts[e], mask)
            dx_perm[rows] = d
            dw1[e] += g1
            dw2[e] += g2
    dx = np.zeros((n, hidden))
    np.add.at(dx, pt, dx_perm)
    dgates = np.zeros((n, plan.k))
    dgates[pt, plan.pair_slots] = dgate_pairs
    if cfg.renormalize:
        raw = np.take_along_axis(r.scores, r.experts, axis=1)
        inner = (dgates * r.gates).sum(axis=1, keepdims=True)
        d_sel = (dgates - inner) / raw.sum(axis=1, keepdims=True)
    else:
        d_sel = dgates
    ds = np.zeros((n, E))
    for s in range(plan.k):
        ds[np.arange(n), r.experts[:, s]] += d_sel[:, s]
    sc = r.scores
    if cfg.gate_fn == "softmax":
        dz = sc * (ds - (ds * sc).sum(axis=1, keepdims=True))
    else:
        dz = ds * sc * (1.0 - sc)
    dwg = None
    if w_g is not None:
        dwg = st.x.T @ dz
        dx = dx + dz @ np.asarray(w_g, dtype=np.float64).T
    sgrads = None
    if shared is not None:
        sdx, sg1, sg2 = expert_backward(u, st.x, st.pres[-1], shared)
        dx = dx + sdx
        sgrads = (sg1, sg2)
    return dx, dz, dwg, dw1, dw2, sgrads


# ----------------------------------------------------------------------------
# seeded inputs (dispatcher.py:197-217, experts.py:66-81)
# ----------------------------------------------------------------------------

def gating_matrix(hidden: int, num_experts: int, seed: int) -> np.ndarray:
    """experts.py:78-81: U(+-1/sqrt(H)) from rng([seed, 0])."""
    b = 1.0 / np.sqrt(hidden)
    return np.random.default_rng([seed, 0]).uniform(-b, b, size=(hidden, num_experts))


def expert_matrices(num_experts: int, hidden: int, ffn: int, seed: int):
    """experts.py:66-75: all W1 then all W2 from rng([seed, 1])."""
    rng = np.random.default_rng([seed, 1])
    b = 1.0 / np.sqrt(hidden)
    w1 = [rng.uniform(-b, b, size=(hidden, ffn)) for _ in range(num_experts)]
    w2 = [rng.uniform(-b, b, size=(ffn, hidden)) for _ in range(num_experts)]
    return w1, w2


def swiglu_matrices(num_experts: int, hidden: int, ffn: int, seed: int):
    """Builder-defined SwiGLU init: gate/up/down U(+-1/sqrt(H)) from
    rng([seed, 4]), w1 = [gate | up]."""
    rng = np.random.default_rng([seed, 4])
    b = 1.0 / np.sqrt(hidden)
    w1, w2 = [], []
    for _ in range(num_experts):
        g = rng.uniform(-b, b, size=(hidden, ffn))
        u = rng.uniform(-b, b, size=(hidden, ffn))
        w1.append(np.concatenate([g, u], axis=1))
        w2.append(rng.uniform(-b, b, size=(ffn, hidden)))
    return w1, w2


def token_rows(n: int, hidden: int, seed: int, stream: int = 2) -> np.ndarray:
    """dispatcher.py:202-204 (stream 2 = x, 3 = upstream)."""
    return np.random.default_rng([seed, stream]).standard_normal((n, hidden))


def rel_err(got, want) -> float:
    """max|got-want| / max|want| -- tests/test_acceptance.py:85-87."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(float(np.abs(want).max()) if want.size else 0.0, 1e-300)
    return float(np.abs(got - want).max() / scale) if want.size else 0.0
