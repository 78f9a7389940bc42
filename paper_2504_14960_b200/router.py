"""Top-k gating and capacity-factor token dropping on the GPU.

Mirrors /root/reference/pkg/src/moefold/router.py: GatingParams :30-74,
RoutingDecision :77-109, compute_gates :127-162, capacity_limit :165-168,
apply_capacity :171-206, gather_full_sequence_decision :209-269, load_stats
:279-301, merge_decisions :304-320.  Arrays are CUDA tensors; the
arithmetic runs in the K1 kernels of libb200moe (router.cu).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np
import torch

from . import _lib as L
from . import kernels as K
from .errors import NumericError, ProtocolError, ValidationError

GATE_SOFTMAX = "softmax"
GATE_SIGMOID = "sigmoid"
DROP_SUBSEQUENCE = "subsequence"
DROP_FULLSEQUENCE = "fullsequence"
PRIORITY_POSITION = "position"
PRIORITY_PROBABILITY = "probability"

GATE_CODES = {GATE_SOFTMAX: L.GATE_SOFTMAX, GATE_SIGMOID: L.GATE_SIGMOID}


def _device_default():
    return torch.device("cuda")


@dataclass
class GatingParams:
    """Router weights plus routing policy (router.py:30-74).  ``w_g`` is
    stored as a CUDA float32 tensor [hidden, experts]."""

    w_g: object
    k: int
    gate_fn: str = GATE_SOFTMAX
    renormalize_topk: bool = False
    capacity_factor: Optional[float] = None
    drop_mode: str = DROP_SUBSEQUENCE
    drop_priority: str = PRIORITY_POSITION

    def __post_init__(self):
        w = self.w_g
        if not isinstance(w, torch.Tensor):
            w = torch.as_tensor(np.asarray(w, dtype=np.float64))
        if w.dim() != 2:
            raise ValidationError("w_g must be 2-D [hidden, experts]", constraint="w_g-2d")
        self.w_g = w
        if not (1 <= self.k <= self.num_experts):
            raise ValidationError(
                f"k must satisfy 1 <= k <= num_experts ({self.num_experts}), got {self.k}",
                constraint="1<=k<=E")
        if self.gate_fn not in GATE_CODES:
            raise ValidationError(f"unknown gate_fn {self.gate_fn!r}", constraint="gate_fn")
        if self.drop_mode not in (DROP_SUBSEQUENCE, DROP_FULLSEQUENCE):
            raise ValidationError(f"unknown drop_mode {self.drop_mode!r}", constraint="drop_mode")
        if self.drop_priority not in (PRIORITY_POSITION, PRIORITY_PROBABILITY):
            raise ValidationError(f"unknown drop_priority {self.drop_priority!r}",
                                  constraint="drop_priority")
        if self.capacity_factor is not None and self.capacity_factor < 1.0:
            raise ValidationError(f"capacity_factor must be >= 1, got {self.capacity_factor}",
                                  constraint="capacity_factor>=1")
        self._dev_cache = {}

    @property
    def num_experts(self) -> int:
        return self.w_g.shape[1]

    @property
    def hidden(self) -> int:
        return self.w_g.shape[0]

    @property
    def dropless(self) -> bool:
        return self.capacity_factor is None

    def device_w_g(self, device=None) -> torch.Tensor:
        """[H, E] fp32 on the device (cached)."""
        device = torch.device(device or _device_default())
        key = ("wg", str(device))
        if key not in self._dev_cache:
            self._dev_cache[key] = self.w_g.to(device=device, dtype=torch.float32).contiguous()
        return self._dev_cache[key]

    def device_w_gT(self, device=None) -> torch.Tensor:
        """[E, H] fp32 on the device (cached) for the backward router term."""
        device = torch.device(device or _device_default())
        key = ("wgT", str(device))
        if key not in self._dev_cache:
            self._dev_cache[key] = self.device_w_g(device).T.contiguous()
        return self._dev_cache[key]

    def device_w_g_parts(self, device=None):
        """W_g as three bf16 parts hi + mid + lo (== W_g exactly) for the
        tensor-core router GEMMs (kernels.router_logits/router_term), cached:
        (w3t [3Ep, H]: rows (part, e), the B operand of x . W_g;
         w6 [H, 6Ep]: column blocks (hi, mid, lo, hi, mid, hi), the B operand
         of dz . W_g^T against dz's (hi, hi, hi, mid, mid, lo))."""
        device = torch.device(device or _device_default())
        key = ("wg_parts", str(device))
        if key not in self._dev_cache:
            w = self.device_w_g(device)
            H, E = w.shape
            Ep = (E + 7) // 8 * 8
            hi = w.to(torch.bfloat16)
            r = w - hi.float()
            mid = r.to(torch.bfloat16)
            lo = (r - mid.float()).to(torch.bfloat16)
            pad = lambda t: torch.nn.functional.pad(t, (0, Ep - E))  # noqa: E731
            hi, mid, lo = pad(hi), pad(mid), pad(lo)
            w3t = torch.cat([hi, mid, lo], dim=1).T.contiguous()
            w6 = torch.cat([hi, mid, lo, hi, mid, hi], dim=1).contiguous()
            self._dev_cache[key] = (w3t, w6)
        return self._dev_cache[key]

    def device_w_g_tc(self, device=None) -> torch.Tensor:
        """B operand of the fused tensor-core router (router_tc.cu): bf16
        [NP, H], rows p * EP + e = part p (hi, mid, lo; hi + mid + lo == W_g
        exactly) of expert e's column, EP = E rounded up to 8/16/32/64, zero
        padded to NP = round_up(3 EP, 16) rows (cached)."""
        device = torch.device(device or _device_default())
        key = ("wg_tc", str(device))
        if key not in self._dev_cache:
            w = self.device_w_g(device)
            H, E = w.shape
            EP = next(c for c in (8, 16, 32, 64, E) if c >= E)
            NP = int(L.load().b200moe_router_fwd_tc_np(E))
            hi = w.to(torch.bfloat16)
            r = w - hi.float()
            mid = r.to(torch.bfloat16)
            lo = (r - mid.float()).to(torch.bfloat16)
            out = torch.zeros((max(NP, 3 * EP), H), dtype=torch.bfloat16, device=device)
            for p, part in enumerate((hi, mid, lo)):
                out[p * EP:p * EP + E] = part.T
            self._dev_cache[key] = out[:NP].contiguous() if NP else out
        return self._dev_cache[key]


@dataclass
class RoutingDecision:
    """Per-token expert assignments (router.py:77-109): ``experts`` int32
    [n,k] best first, ``gates`` fp32 [n,k], ``kept`` bool [n,k], ``positions``
    int64 [n] (host or device), ``scores`` fp32 [n,E] when available."""

    experts: torch.Tensor
    gates: torch.Tensor
    kept: torch.Tensor
    positions: torch.Tensor
    scores: Optional[torch.Tensor] = None
    gates_f64: Optional[torch.Tensor] = None

    def __post_init__(self):
        # reference callers build decisions from numpy arrays (router.py:77-109);
        # they move to the device once here, device tensors pass through
        dev = next((t.device for t in (self.experts, self.gates, self.kept)
                    if isinstance(t, torch.Tensor) and t.is_cuda), None) or _device_default()

        def conv(v, dtype):
            if v is None or isinstance(v, torch.Tensor):
                return v
            return torch.as_tensor(np.asarray(v)).to(dev, dtype).contiguous()

        self.experts = conv(self.experts, torch.int32)
        self.gates = conv(self.gates, torch.float32)
        self.kept = conv(self.kept, torch.bool)
        self.scores = conv(self.scores, torch.float32)
        if not isinstance(self.positions, torch.Tensor):
            self.positions = torch.as_tensor(np.asarray(self.positions), dtype=torch.int64)

    @property
    def n_tokens(self) -> int:
        return self.experts.shape[0]

    @property
    def k(self) -> int:
        return self.experts.shape[1]

    def copy(self) -> "RoutingDecision":
        c = lambda t: None if t is None else t.clone()  # noqa: E731
        return RoutingDecision(c(self.experts), c(self.gates), c(self.kept), c(self.positions),
                               c(self.scores), c(self.gates_f64))


def nonfinite_error(x: Optional[torch.Tensor], params: GatingParams, suffix: str = "") -> NumericError:
    """The router.py:141-144 error for a step whose router flagged non-finite
    logits: the token block unless it is finite, then the gating weights
    (only evaluated on the error path)."""
    if x is not None and bool(torch.isfinite(x).all()) and \
            not bool(torch.isfinite(params.device_w_g(x.device)).all()):
        return NumericError("gating weights contain non-finite values" + suffix)
    return NumericError("token block contains non-finite values" + suffix)


def routing_from_logits(logits: torch.Tensor, params: GatingParams, positions=None,
                        want_f64: bool = False, status: Optional[torch.Tensor] = None) -> RoutingDecision:
    """Scores, top-k and gates from fp32 logits (router.py:146-162).  A token
    with non-finite logits sets bit 0 of ``status`` and gets the placeholder
    routing 0..k-1."""
    n = logits.shape[0]
    scores, idx, gates, g64 = K.router_topk(
        logits.contiguous(), params.k, GATE_CODES[params.gate_fn], params.renormalize_topk,
        want_f64=want_f64 or params.drop_priority == PRIORITY_PROBABILITY, status=status)
    if positions is None:
        positions = torch.arange(n, dtype=torch.int64)
    else:
        positions = torch.as_tensor(positions, dtype=torch.int64)
        if tuple(positions.shape) != (n,):
            raise ValidationError("positions must have one entry per token", constraint="positions")
    kept = torch.ones((n, params.k), dtype=torch.bool, device=logits.device)
    return RoutingDecision(idx, gates, kept, positions, scores, g64)


def compute_gates(x, params: GatingParams, positions=None, *, check: bool = True) -> RoutingDecision:
    """Score a token block and select each token's top-k experts (router.py:127-162)."""
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(np.asarray(x, dtype=np.float64), dtype=torch.float32)
    if not x.is_cuda:
        x = x.to(_device_default())
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.float()
    x = x.contiguous()
    if x.dim() != 2 or x.shape[1] != params.hidden:
        raise ValidationError(f"token block shape {tuple(x.shape)} incompatible with w_g "
                              f"{tuple(params.w_g.shape)}", constraint="x-shape")
    status = torch.zeros((1,), dtype=torch.int32, device=x.device)
    if x.dtype == torch.bfloat16 and K.router_fwd_supported(x, params.num_experts):
        # fused tensor-core router (router_tc.cu): x read once
        _, scores, idx, gates, g64 = K.router_fwd(
            x, params.device_w_g_tc(x.device), params.num_experts, params.k,
            GATE_CODES[params.gate_fn], params.renormalize_topk, status,
            want_f64=params.drop_priority == PRIORITY_PROBABILITY)
        n = x.shape[0]
        pos = torch.arange(n, dtype=torch.int64) if positions is None else positions
        dec = RoutingDecision(idx, gates, torch.ones((n, params.k), dtype=torch.bool, device=x.device),
                              torch.as_tensor(pos, dtype=torch.int64), scores, g64)
        if dec.positions.shape != (n,):
            raise ValidationError("positions must have one entry per token", constraint="positions")
    else:
        logits = K.router_logits(x, params.device_w_g(x.device))
        dec = routing_from_logits(logits, params, positions, status=status)
    # router.py:141-144: one host read of the flag the kernels raised (no
    # separate pass over x)
    if check and int(status.item()) & 1:
        raise nonfinite_error(x, params)
    return dec


def capacity_limit(capacity_factor: float, l_scope: int, num_experts: int) -> int:
    """floor(CF * L / E), at least one (router.py:165-168; no k factor)."""
    return max(1, math.floor(capacity_factor * l_scope / num_experts))


def _monotone(positions: torch.Tensor) -> bool:
    p = positions.cpu() if positions.is_cuda else positions
    return p.numel() < 2 or bool((p[1:] > p[:-1]).all())


def kept_mask(decision: RoutingDecision, l_scope: int, num_experts: int,
              params: GatingParams, cap: Optional[int] = None,
              sorted_positions: bool = False) -> torch.Tensor:
    """Capacity drop flags as a uint8 [n,k] device tensor (router.py:171-206).
    ``cap`` overrides capacity_limit(l_scope, num_experts) (virtual experts);
    ``sorted_positions`` skips the host monotonicity check."""
    dev = decision.experts.device
    n, k = decision.experts.shape
    kept_in = decision.kept.to(torch.uint8).contiguous()
    if params.dropless:
        return kept_in
    if cap is None:
        cap = capacity_limit(params.capacity_factor, l_scope, num_experts)
    idx = decision.experts.contiguous()
    if params.drop_priority == PRIORITY_POSITION:
        order = None
        if not sorted_positions and not _monotone(decision.positions):
            order = torch.argsort(decision.positions.cpu(), stable=True).to(torch.int32).to(dev)
        plan = K.dispatch_plan(idx, decision.gates, num_experts, cap=cap, kept_in=kept_in,
                               order=order, want_perm_gates=False)
        return plan.kept
    g64 = decision.gates_f64 if decision.gates_f64 is not None else decision.gates.double()
    plan0 = K.dispatch_plan(idx, decision.gates, num_experts, cap=0, kept_in=kept_in,
                            want_perm_gates=False)
    pos = decision.positions.to(dev, torch.int64)
    kept = K.capacity_by_gate(plan0, g64.contiguous(), pos, cap)
    return kept & kept_in


def apply_capacity(decision: RoutingDecision, l_scope: int, num_experts: int,
                   params: GatingParams) -> RoutingDecision:
    """Drop pairs exceeding per-expert capacity within one scope (router.py:171-206)."""
    if params.dropless:
        return decision
    if params.capacity_factor < 1.0:
        raise ValidationError("capacity_factor must be >= 1", constraint="capacity_factor>=1")
    out = decision.copy()
    out.kept = kept_mask(decision, l_scope, num_experts, params).bool()
    return out


def gather_full_sequence_decision(ctx, group, local: RoutingDecision, seq_len: int,
                                  num_experts: int, params: GatingParams, check: bool = True,
                                  slots: Optional[int] = None, status: Optional[torch.Tensor] = None,
                                  want_global: bool = True
                                  ) -> Tuple[Optional[RoutingDecision], RoutingDecision]:
    """Capacity per full sequence across the ranks sharding it (router.py:209-269).

    Device-native: every member's pairs travel as int64 keys -- segment
    (sequence x expert) and position, plus the float64 gate under probability
    priority -- through a fixed-size all-gather (``slots`` tokens per member,
    padded; no sizes cross the host), are sorted on the device into admission
    order (stable sorts: position, [gate descending,] segment), and one
    kernel (b200moe_fullseq_capacity) gives every pair its rank inside its
    segment, keeps it iff rank < cap, and writes the flags back to the pairs'
    slots.  Nothing in the layer path synchronises with the host; the
    duplicate-position check (router.py:245-246) is a status bit (``status``,
    raised by moe_forward) -- or, standalone with ``check``, a host read.
    ``slots`` defaults to the group's largest block, agreed with one host
    exchange.  The global decision (union of the group's pairs in position
    order) is built only when ``want_global``."""
    n, k = local.experts.shape
    E = num_experts
    group = tuple(group)
    me = group.index(ctx.rank)
    dev = local.experts.device
    if slots is None:
        slots = max(int(v) for v in ctx.meta(group, n).values())
    oversize = n > slots
    if oversize:
        if status is None:
            raise ValidationError(f"token block of {n} rows exceeds the {slots} full-sequence gather slots",
                                  constraint="fullseq-slots")
        # the layer path: take part in the group's gather with no pairs and
        # fail the step through the status word (bit 2) on every rank
        status.bitwise_or_(4)
    S = slots * k
    pos_h = local.positions
    if pos_h.is_cuda:
        pos = pos_h.to(torch.int64)
    else:
        pos = pos_h.to(torch.int64).pin_memory().to(dev, non_blocking=True)
    pad = torch.iinfo(torch.int64).max
    seg = torch.full((S,), pad, dtype=torch.int64, device=dev)
    ppos = torch.full((S,), pad, dtype=torch.int64, device=dev)
    if n and not oversize:
        seg[:n * k] = ((pos // seq_len)[:, None] * E + local.experts.to(torch.int64)).reshape(-1)
        ppos[:n * k] = pos.repeat_interleave(k)
    # the reference's wire record: (pos, slot, expert, gate) rows of width 4
    ctx.account(group, "all_gather_v", 4, n * k)
    all_seg = ctx.all_gather_fixed(group, seg).view(-1)
    all_pos = ctx.all_gather_fixed(group, ppos).view(-1)
    by_pos = torch.sort(all_pos, stable=True).indices
    order = by_pos
    prob = params.drop_priority == PRIORITY_PROBABILITY
    g64 = None
    if prob or want_global:
        g = local.gates_f64 if local.gates_f64 is not None else local.gates.double()
        gp = torch.full((S,), float("-inf"), dtype=torch.float64, device=dev)
        if n and not oversize:
            gp[:n * k] = g.reshape(-1)
        g64 = ctx.all_gather_fixed(group, gp).view(-1)
    if prob:
        order = order[torch.sort(g64[order], descending=True, stable=True).indices]
    order = order[torch.sort(all_seg[order], stable=True).indices]
    cap = capacity_limit(params.capacity_factor, seq_len, E)
    own_status = status if status is not None else torch.zeros((1,), dtype=torch.int32, device=dev)
    kept_slot = K.fullseq_capacity(all_seg[order].contiguous(), order.contiguous(), cap, k,
                                   pos_by_pos=all_pos[by_pos].contiguous(), status=own_status)
    if status is None and check and int(own_status.item()) & 8:
        raise ProtocolError("full-sequence gather: duplicate token positions across shards")
    out = local.copy()
    if oversize:
        out.kept = torch.zeros((n, k), dtype=torch.bool, device=dev)
    else:
        out.kept = kept_slot.view(len(group), S)[me, :n * k].view(n, k).bool()
    global_dec = None
    if want_global:
        # the group's pairs in position order (sizes read on the host: API use only)
        valid = all_pos[by_pos] != pad
        idx = by_pos[valid]
        # a token's k pairs share its position and sit in slot order (t*k + s),
        # so the stable position sort keeps them adjacent and best-first
        tok = idx.view(-1, k)
        gg = g64[tok]
        global_dec = RoutingDecision((all_seg[tok] % E).to(torch.int32).contiguous(), gg.float(),
                                     kept_slot[tok].bool(), all_pos[tok[:, 0]].cpu(), None, gg.contiguous())
    return global_dec, out


@dataclass(frozen=True)
class LoadStats:
    counts: np.ndarray
    imbalance: float
    aux_loss: float


def load_stats(decision: RoutingDecision, num_experts: int) -> LoadStats:
    """Kept pairs per expert, imbalance, Switch aux loss (router.py:279-301):
    one deterministic reduction kernel (router_stats), one host read."""
    n = decision.n_tokens
    scores = None if decision.scores is None else decision.scores.float().contiguous()
    counts_d, top1_d, psum_d = K.router_stats(decision.experts.contiguous(), decision.kept, scores,
                                              num_experts)
    counts = counts_d.cpu().numpy().astype(np.int64)
    mean = counts.sum() / num_experts
    imbalance = float(counts.max() / mean) if mean > 0 else float("nan")
    if scores is None or n == 0:
        aux = float("nan")
    else:
        f = top1_d.double() / n
        p = psum_d / n
        aux = float(num_experts * torch.dot(f, p))
    return LoadStats(counts=counts, imbalance=imbalance, aux_loss=aux)


def merge_decisions(decisions) -> RoutingDecision:
    """Concatenate per-rank decisions ordered by global position (router.py:304-320)."""
    dev = decisions[0].experts.device
    cat = lambda name: torch.cat([getattr(d, name).to(dev) for d in decisions])  # noqa: E731
    positions = cat("positions")
    order = torch.argsort(positions, stable=True)
    scores = None
    if all(d.scores is not None for d in decisions):
        scores = cat("scores")[order]
    return RoutingDecision(cat("experts")[order], cat("gates")[order], cat("kept")[order],
                           positions[order], scores)
