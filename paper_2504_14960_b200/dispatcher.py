"""Token-level dispatch: the MoE layer forward/backward on B200.

Mirrors /root/reference/pkg/src/moefold/dispatcher.py (TokenBlock :44-59,
DispatchPlan :62-93, build_dispatch_plan :96-131, permute :134-142,
unpermute_combine :145-157, token_partition :160-194, fabricate_* :197-217,
ForwardContext :220-229, BackwardResult :232-236, moe_forward :246-384,
moe_backward :387-510).

Per rank (SPMD), forward:
  K1 router (logits, top-k, capacity + plan as one counting sort)
  one rank (EP = ETP = 1): K2 permute straight into the padded GEMM layout
    -> K3 grouped FFN -> K2 gate-weighted combine
  several ranks, bf16 (default): device-side exchange over NVLink peer
    memory (peer.py): counts pushed to every member, receive layouts derived
    on the device, token rows pushed into the owners' buffers (the ETP
    all-gather folded in) -> K3 grouped FFN whose epilogue stores each
    output row straight back into its sender's layout (the return
    all-to-all and, per ETP member block, the reduce-scatter) -> combine
  NCCL path (fp32 parity mode, B200MOE_EP_EXCHANGE=nccl): counts exchanged
    once, all_to_all_single into the padded expert-major layout, ETP
    all-gather-v / reduce-scatter-v as P2P, return all-to-all, combine
Backward mirrors it, then the router backward and the dW_g all-reduce over
the world (expert grads over EDP).
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from . import _lib as L
from . import experts as X
from . import gemm_tc
from . import kernels as K
from .collectives import LocalWorld, RankContext
from .errors import NumericError, ProtocolError, ValidationError
from .router import (DROP_FULLSEQUENCE, GATE_CODES, PRIORITY_PROBABILITY, GatingParams,
                     RoutingDecision, capacity_limit, gather_full_sequence_decision,
                     kept_mask, nonfinite_error, routing_from_logits)
from .topology import (GroupSets, ParallelTopology, check_pp_consistency,
                       generate_parallel_groups, sequence_group)

ALIGN = K.GEMM_ALIGN


@dataclass
class TokenBlock:
    """One rank's flattened token rows plus their global coordinates."""

    values: object  # [rows, hidden] tensor (CUDA) or array
    positions: object  # [rows] global token ids

    def __post_init__(self):
        v = self.values
        if not isinstance(v, torch.Tensor):
            v = torch.as_tensor(np.asarray(v, dtype=np.float64))
        if v.dim() != 2:
            raise ValidationError("token block must be 2-D", constraint="block-2d")
        p = torch.as_tensor(np.asarray(self.positions) if not isinstance(self.positions, torch.Tensor)
                            else self.positions, dtype=torch.int64).cpu()
        if tuple(p.shape) != (v.shape[0],):
            raise ValidationError("positions must have one entry per row",
                                  constraint="positions-per-row")
        self.values = v
        self.positions = p


@dataclass
class DispatchPlan:
    """Permutation and counts of one rank's exchange (dispatcher.py:62-93).

    ``permutation``/``send_counts``/``gates`` follow the reference exactly
    (host views are materialised lazily).  Device fields drive the kernels:
    ``send_row``/``gemm_row`` [n,k] map each kept pair to its row in send order
    / in the padded expert-major layout (-1 when dropped)."""

    dev: K.PlanTensors
    n_tokens: int
    k: int
    ep_size: int
    local_experts: int
    pair_gates: Optional[torch.Tensor] = None  # [n,k] fp32 device
    # rows received per (EP sender, local expert) in the dispatch all-to-all
    # (dispatcher.py:313-316): a device tensor or host array, read lazily
    recv_src: object = None
    _host: Dict = field(default_factory=dict, repr=False)

    @property
    def recv_counts(self) -> Optional[np.ndarray]:
        if self.recv_src is None:
            return None
        if "recv" not in self._host:
            r = self.recv_src
            r = r.detach().cpu().numpy() if isinstance(r, torch.Tensor) else np.asarray(r)
            self._host["recv"] = r.astype(np.int64).reshape(self.ep_size, self.local_experts)
        return self._host["recv"]

    @recv_counts.setter
    def recv_counts(self, value):
        self.recv_src = value
        self._host.pop("recv", None)

    def _offsets(self) -> np.ndarray:
        if "off" not in self._host:
            self._host["off"] = self.dev.offsets.cpu().numpy().astype(np.int64)
        return self._host["off"]

    @property
    def n_send(self) -> int:
        return int(self._offsets()[-1])

    @property
    def permutation(self) -> np.ndarray:
        return self.dev.perm[: self.n_send].cpu().numpy()

    @property
    def send_counts(self) -> np.ndarray:
        return self.dev.counts.cpu().numpy().astype(np.int64).reshape(self.ep_size, self.local_experts)

    @property
    def gates(self) -> np.ndarray:
        return self.dev.perm_gates[: self.n_send].cpu().numpy()

    @property
    def kept(self) -> torch.Tensor:
        return self.dev.kept.bool()

    @property
    def pair_tokens(self) -> np.ndarray:
        return self.permutation // self.k

    @property
    def pair_slots(self) -> np.ndarray:
        return self.permutation % self.k

    @property
    def restore(self) -> np.ndarray:
        return self.permutation


def build_dispatch_plan(decision: RoutingDecision, ep_group_size: int,
                        local_expert_count: int) -> DispatchPlan:
    """Order a rank's kept pairs for dispatch (dispatcher.py:96-131): one
    stable counting sort by global expert id on the device."""
    E = ep_group_size * local_expert_count
    idx = decision.experts.to(torch.int32).contiguous()
    if idx.numel() and int(idx.max()) >= E:
        raise ValidationError(f"expert id {int(idx.max())} out of range for {E} experts",
                              constraint="expert<E")
    n, k = idx.shape
    plan = K.dispatch_plan(idx, decision.gates.float().contiguous(), E, cap=0,
                           kept_in=decision.kept.to(torch.uint8).contiguous())
    return DispatchPlan(plan, n, k, ep_group_size, local_expert_count,
                        pair_gates=decision.gates.float().contiguous())


def permute(values, plan: DispatchPlan) -> torch.Tensor:
    """Gather token rows into send order (dispatcher.py:134-142)."""
    v = values if isinstance(values, torch.Tensor) else torch.as_tensor(np.asarray(values))
    v = v.to(plan.dev.send_row.device).contiguous()
    if v.dtype not in (torch.float32, torch.bfloat16):
        v = v.float()
    if v.shape[0] != plan.n_tokens:
        raise ValidationError(f"block has {v.shape[0]} rows, plan expects {plan.n_tokens}",
                              constraint="rows==plan.n_tokens")
    out = K.permute(v, plan.dev.send_row, plan.n_send)
    return out[: plan.n_send]


def unpermute_combine(rows, plan: DispatchPlan, hidden: int) -> torch.Tensor:
    """Gate-weighted scatter back to token order (dispatcher.py:145-157)."""
    r = rows if isinstance(rows, torch.Tensor) else torch.as_tensor(np.asarray(rows))
    r = r.to(plan.dev.send_row.device).contiguous()
    if r.dtype not in (torch.float32, torch.bfloat16):
        r = r.float()
    if r.shape[0] != plan.n_send:
        raise ValidationError(f"{r.shape[0]} returned rows for {plan.n_send} plan slots",
                              constraint="rows==plan-slots")
    if r.shape[0] == 0:
        r = torch.zeros((1, hidden), dtype=r.dtype, device=r.device)
    return K.combine(r, plan.dev.send_row, plan.n_tokens, gates=plan.pair_gates)


def token_partition(topology: ParallelTopology, seq_len: int, batch: int) -> List[np.ndarray]:
    """Global token ids per rank: sequences dealt to DP replicas in contiguous
    batches, each split over TP x CP context-major (dispatcher.py:160-194)."""
    if topology.pp != 1:
        raise ValidationError("token partitioning requires pp == 1", constraint="pp==1")
    shards = topology.tp * topology.cp
    if seq_len % shards:
        raise ValidationError(f"seq_len={seq_len} is not divisible by tp*cp={shards}",
                              constraint="tp*cp|seq_len")
    if batch % topology.dp:
        raise ValidationError(f"batch={batch} is not divisible by dp={topology.dp}",
                              constraint="dp|batch")
    chunk = seq_len // shards
    per = batch // topology.dp
    out = []
    for rank in range(topology.world_size):
        t, c, d, _ = topology.attn_coords(rank)
        shard = c * topology.tp + t
        starts = (d * per + np.arange(per)) * seq_len + shard * chunk
        out.append((starts[:, None] + np.arange(chunk)[None, :]).reshape(-1).astype(np.int64))
    return out


def fabricate_token_blocks(topology, seq_len, batch, hidden, seed, dtype=torch.float32, device=None):
    """Seeded stand-in for attention outputs (dispatcher.py:197-207): x ~ N(0,1)
    from rng([seed, 2]); blocks hold device tensors of ``dtype``."""
    x = np.random.default_rng([seed, 2]).standard_normal((batch * seq_len, hidden))
    parts = token_partition(topology, seq_len, batch)
    dev = torch.device(device or "cuda")
    blocks = [TokenBlock(torch.as_tensor(x[p]).to(dev, dtype), p) for p in parts]
    return x, blocks


def fabricate_upstream(topology, seq_len, batch, hidden, seed, dtype=torch.float32, device=None):
    """dispatcher.py:210-217 (rng([seed, 3]))."""
    u = np.random.default_rng([seed, 3]).standard_normal((batch * seq_len, hidden))
    parts = token_partition(topology, seq_len, batch)
    dev = torch.device(device or "cuda")
    return u, [torch.as_tensor(u[p]).to(dev, dtype) for p in parts]


@dataclass
class ForwardContext:
    world: object
    topology: ParallelTopology
    params: GatingParams
    weights_map: Dict[Tuple[int, int], X.ExpertWeights]
    groups: GroupSets
    per_rank: List[dict] = field(default_factory=list)

    def check(self) -> None:
        """Wait for the step's device status and raise what it flagged
        (NumericError / ProtocolError / ValidationError, router.py:141-144):
        the explicit synchronisation point; moe_forward / moe_backward raise
        without waiting when the status has already landed, and the next
        moe_forward on the world raises a pending one."""
        _check_step(self, block=True)
        if self.world.__dict__.get("_b200moe_pending") is self:
            del self.world.__dict__["_b200moe_pending"]


@dataclass
class BackwardResult:
    input_grads: List[Optional[torch.Tensor]]
    w_g_grad: torch.Tensor
    expert_grads: Dict[Tuple[int, int], Tuple[List[torch.Tensor], List[torch.Tensor]]]
    # builder-defined shared expert: (dW1 [H, 2F_s], dW2 [F_s, H]) summed over ranks
    shared_grads: Optional[Tuple[torch.Tensor, torch.Tensor]] = None


# =========================================================== rank program
@dataclass
class LayerGroups:
    ep: Tuple[int, ...]
    etp: Tuple[int, ...]
    edp: Tuple[int, ...]
    world: Tuple[int, ...]
    seq: Tuple[int, ...]
    xch: Tuple[int, ...] = ()  # EP x ETP block (member = ep_idx * etp + etp_idx)


@dataclass
class ExchangePlan:
    """Host-side sizes of one rank's EP all-to-all-v and ETP gather, computed
    from the all-gathered per-expert counts (the one host sync of the layer).

    A rank's send buffer is its padded per-global-expert layout; the block it
    receives from sender s is s's chunks for this rank's local experts, each
    padded to ``align`` rows.  With ETP the gathered buffer is member-major."""

    send_splits: List[int]  # rows to each EP peer (padded)
    recv_splits: List[int]  # rows from each EP peer (padded)
    recv_padded: np.ndarray  # [ep, L] padded rows of (sender, local expert) segments
    recv_counts: np.ndarray  # [ep, L] real rows of those segments
    block_off: np.ndarray  # [etp+1] member block offsets in the gathered buffer
    group_off: List[int]  # [G+1] GEMM group offsets (member, sender, le) in the gathered buffer
    group_expert: List[int]  # [G] local expert of each group


def _pad(c, align):
    return (np.asarray(c, dtype=np.int64) + align - 1) // align * align


def exchange_plan(counts: np.ndarray, ep_pos: int, L_: int, etp_recv: Optional[np.ndarray] = None,
                  align: int = ALIGN) -> ExchangePlan:
    """Pure host arithmetic (tested on CPU).

    counts [ep, ep*L]: row s = EP member s's kept pairs per global expert of
    this EP group.  etp_recv [etp, ep*L] (None when ETP = 1): every ETP
    member's ``recv_padded`` flattened, in ETP-rank order."""
    counts = np.asarray(counts, dtype=np.int64)
    ep = counts.shape[0]
    padded = _pad(counts, align)
    send_splits = [int(padded[ep_pos, d * L_:(d + 1) * L_].sum()) for d in range(ep)]
    recv_padded = padded[:, ep_pos * L_:(ep_pos + 1) * L_]
    recv_counts = counts[:, ep_pos * L_:(ep_pos + 1) * L_]
    recv_splits = [int(recv_padded[s].sum()) for s in range(ep)]
    members = [recv_padded.reshape(-1)] if etp_recv is None else [np.asarray(r).reshape(-1) for r in etp_recv]
    block_off = np.concatenate(([0], np.cumsum([int(m.sum()) for m in members]))).astype(np.int64)
    group_off, group_expert = [], []
    for mi, m in enumerate(members):
        off = block_off[mi] + np.concatenate(([0], np.cumsum(m)))[:-1]
        group_off.extend(int(o) for o in off)
        group_expert.extend(i % L_ for i in range(m.size))
    group_off.append(int(block_off[-1]))
    return ExchangePlan(send_splits, recv_splits, recv_padded, recv_counts, block_off, group_off,
                        group_expert)


# ----------------------------------------------------------- step status
# Failures the device detects (router.py:141-144 non-finite inputs, a peer
# buffer too small for the block, a peer whose step failed) are bits of a
# per-rank int32 status word instead of blocking host checks: the router and
# exchange kernels set them, the word is copied to pinned host memory right
# after the router / the dispatch barrier, and moe_forward raises after
# waiting for that early point of the step only (the GEMMs stay queued).
ST_NONFINITE, ST_PEER_ABORT, ST_OVERSIZE, ST_DUPLICATE, ST_RECV_OVERFLOW = 1, 2, 4, 8, 16
_STATUS: Dict[tuple, tuple] = {}
_SIDE: Dict[tuple, torch.cuda.Stream] = {}
# measured neutral at 4 GPUs (C4: 36.4 vs 36.0 ms/step): the barrier wait it
# fills is the slowest GPU's skew, which the slowest GPU itself cannot hide
_SIDE_SHARED = os.environ.get("B200MOE_SHARED_SIDE", "0") == "1"


def _overlap_fits(ctx) -> bool:
    """The overlapped push keeps a side push and a landing barrier in flight
    beside a persistent GEMM per rank; ranks emulated on one GPU share its
    SMs, and measured, 8 of them can starve each other's side pushes into a
    barrier timeout (tests/test_gpu_device_barrier.py).  Allow it with at
    most 4 ranks per device (one process per GPU always fits)."""
    world = getattr(ctx, "world", None)
    if world is None or not hasattr(world, "device_of") or not hasattr(world, "n_ranks"):
        return True
    me = world.device_of(ctx.rank)
    return sum(1 for r in range(world.n_ranks) if world.device_of(r) == me) <= 4


def _side_stream(device, main) -> "torch.cuda.Stream":
    """One side stream per compute stream (ranks of a LocalWorld that share a
    GPU each have their own)."""
    key = (str(device), main.cuda_stream)
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=device)
    return _SIDE[key]


def _status_slot(device, rank: int, tag=0):
    key = (str(device), rank, tag)
    slot = _STATUS.get(key)
    if slot is None:
        slot = (torch.zeros((1,), dtype=torch.int32, device=device),
                torch.zeros((1,), dtype=torch.int32).pin_memory(),
                torch.zeros((1,), dtype=torch.int32, device=device))  # scratch (unchecked steps)
        _STATUS[key] = slot
    return slot


def _raise_status(bits: int, what: str = "") -> None:
    if bits & ST_NONFINITE:
        raise NumericError(f"token block contains non-finite values{what}")
    if bits & ST_DUPLICATE:
        raise ProtocolError(f"full-sequence gather: duplicate token positions across shards{what}")
    if bits & ST_OVERSIZE:
        raise ValidationError(f"token block exceeds the peer buffers / full-sequence gather slots sized on "
                              f"first use{what}: pass peer_tokens >= the largest block on first use",
                              constraint="peer-capacity")
    if bits & ST_RECV_OVERFLOW:
        raise ProtocolError(f"this step's routing overflows the peer receive buffers{what}: raise "
                            "peer_capacity (None = worst case) or rebalance the router")
    if bits & ST_PEER_ABORT:
        raise ProtocolError(f"a member of the expert-parallel exchange failed this step{what}")


class RankLayer:
    """Everything one rank needs to run the layer forward and backward."""

    def __init__(self, params: GatingParams, weights: X.ExpertWeights, topology: ParallelTopology,
                 groups: LayerGroups, rank: int, dtype, device, seq_len=None, check=False,
                 shared: Optional[X.ExpertWeights] = None, pad_to_capacity: bool = False,
                 exchange: Optional[str] = None, peer_tokens: Optional[int] = None, peer_tag=0,
                 peer_capacity: Optional[float] = None):
        self.shared_pk = None if shared is None else shared.packed(dtype, device)
        # pad-to-capacity (BASELINE C3): every expert segment holds exactly
        # round_up(cap, ALIGN) rows, so all exchange sizes are static and the
        # layer never synchronises with the host.  Sub-sequence dropping only
        # (the per-rank capacity bounds every segment).
        self.pad_to_capacity = pad_to_capacity
        # NCCL path: overlap the EP all-to-all with the FFN of the rank's own
        # rows (B200MOE_OVERLAP=0 selects the serial exchange)
        self.overlap = os.environ.get("B200MOE_OVERLAP", "1") != "0"
        self.params = params
        self.topo = topology
        self.g = groups
        self.rank = rank
        self.dtype = dtype
        self.device = device
        self.seq_len = seq_len
        self.check = check
        self.E = params.num_experts
        self.k = params.k
        self.L = self.E // topology.ep
        self.w = weights
        self.pk = weights.packed(dtype, device)
        self.wg = params.device_w_g(device)
        self.wgT = params.device_w_gT(device)
        # bf16 tokens: the three router GEMMs on the tensor cores against the
        # exact bf16 parts of W_g (B200MOE_ROUTER_TC=0: CUDA-core kernels)
        self.wg_parts = None
        if dtype == torch.bfloat16 and os.environ.get("B200MOE_ROUTER_TC", "1") != "0":
            self.wg_parts = params.device_w_g_parts(device)
        self.single = len(groups.ep) == 1 and len(groups.etp) == 1
        # EP / ETP exchange: device-side over NVLink peer memory (bf16; the
        # return direction is the tensor-core GEMM's scatter epilogue), or
        # NCCL (B200MOE_EP_EXCHANGE=nccl, and the fp32 parity mode)
        self.peer_tokens = peer_tokens
        self.peer_capacity = peer_capacity
        self.peer_tag = peer_tag
        want = exchange or os.environ.get("B200MOE_EP_EXCHANGE", "peer")
        if want not in ("peer", "nccl"):
            raise ValidationError(f"unknown EP exchange {want!r}", constraint="exchange")
        self.use_peer = (want == "peer" and not self.single and 1 < len(groups.xch) <= 32
                         and dtype == torch.bfloat16 and self.k <= 8 and gemm_tc.available()
                         and self.pk.hidden % 8 == 0 and self.pk.ffn % 8 == 0)
        # peer path, B200MOE_PUSH_OVERLAP=1: the NVLink part of each push runs
        # on a side stream beside the first GEMM over the rank's own rows
        # (bit-identical).  Off by default: measured neutral to negative in the
        # layer at 4 GPUs (-4 to +2 % across C2-C5)
        self.push_overlap = (self.use_peer and X.split_ok(self.pk, dtype)
                             and os.environ.get("B200MOE_PUSH_OVERLAP", "0") == "1")
        # step status (see _status_slot): the router writes bit 0 into the
        # checked word only when inputs are validated
        self.status, self.status_host, self.scratch = _status_slot(device, rank, peer_tag)
        self.status_event = None

    # ------------------------------------------------------- shared expert
    # Builder-defined (no reference): a dense FFN over every token whose
    # output is added to the routed combine (Qwen2-57B-A14B, BASELINE C4).
    # One GEMM group spanning all T rows; the ragged tail tile reads past
    # the buffer end, which TMA zero-fills.
    def _shared_forward(self, x, saved):
        if self.shared_pk is None:
            return None
        T = x.shape[0]
        goff = K._single_group(T, x.device)
        pre, h, y = X.ffn_forward(x, goff, 1, None, self.shared_pk, T)
        saved.update(s_pre=pre, s_h=h, s_goff=goff)
        return y

    def _shared_backward(self, u, sv):
        if self.shared_pk is None:
            return None, None
        T = u.shape[0]
        dx, dw1, dw2 = X.ffn_backward(u, sv["x"], sv["s_pre"], sv["s_h"], sv["s_goff"], 1, None,
                                      self.shared_pk, T)
        return dx, (dw1, dw2)

    # With the peer exchange the shared expert's GEMMs run on a side stream
    # while the compute stream waits in the cross-GPU barrier after the routed
    # GEMMs (that wait is the other GPUs' skew and their last scatter stores):
    # the side work is released by an event recorded right after the routed
    # GEMMs, so it never takes SMs from them, and the combine waits for it.
    # Opt-in (B200MOE_SHARED_SIDE=1): measured neutral, see _SIDE_SHARED.
    def _on_side(self, fn, *args):
        main = torch.cuda.current_stream()
        side = _side_stream(self.device, main)
        go = torch.cuda.Event()
        go.record(main)
        side.wait_event(go)
        with torch.cuda.stream(side):
            out = fn(*args)
            done = torch.cuda.Event()
            done.record(side)
        return out, done, main

    def _shared_forward_side(self, x, saved):
        if self.shared_pk is None or not _SIDE_SHARED:
            return self._shared_forward(x, saved), None
        y, done, main = self._on_side(self._shared_forward, x, saved)
        for t in (y, saved["s_pre"], saved["s_h"]):  # made on the side stream, used on the main one
            t.record_stream(main)
        return y, done

    def _shared_backward_side(self, u, sv):
        if self.shared_pk is None or not _SIDE_SHARED:
            return None
        (dx, grads), done, main = self._on_side(self._shared_backward, u, sv)
        for t in (dx,) + tuple(grads):
            t.record_stream(main)
        return dx, grads, done

    # ---------------------------------------------------------------- fwd
    def forward(self, ctx: Optional[RankContext], x: torch.Tensor, positions: torch.Tensor) -> Tuple[torch.Tensor, dict]:
        p = self.params
        T, H = x.shape
        x = x.to(self.device, self.dtype).contiguous()
        self.status.zero_()
        self.status_event = None
        rst = self.status if self.check else self.scratch
        want64 = p.drop_priority == PRIORITY_PROBABILITY
        if self.wg_parts is not None and K.router_fwd_supported(x, self.E):
            # fused: x read once by TMA, logits on the tensor cores, softmax /
            # sigmoid and top-k in the epilogue (router_tc.cu)
            logits, scores, idx, gates, g64 = K.router_fwd(
                x, p.device_w_g_tc(self.device), self.E, self.k, GATE_CODES[p.gate_fn],
                p.renormalize_topk, rst, want_f64=want64)
            kept = torch.ones((T, self.k), dtype=torch.bool, device=x.device)
            dec = RoutingDecision(idx, gates, kept, torch.as_tensor(positions, dtype=torch.int64),
                                  scores, g64)
        else:
            logits = K.router_logits(x, self.wg, parts=self.wg_parts)
            dec = routing_from_logits(logits, p, positions, status=rst)
        return self.forward_routed(ctx, x, dec, logits)

    def _mark_status(self):
        """Copy the status word to pinned host memory at this point of the
        stream (read by moe_forward via check_status)."""
        self.status_host.copy_(self.status, non_blocking=True)
        self.status_event = torch.cuda.Event()
        self.status_event.record()

    def check_status(self, what: str = "") -> None:
        if self.status_event is None:
            return
        self.status_event.synchronize()
        _raise_status(int(self.status_host[0]), what)

    def forward_routed(self, ctx, x, dec: RoutingDecision, logits=None):
        p = self.params
        T, H = x.shape
        E, k = self.E, self.k
        # ---- capacity (router.py:171-269) ----
        if not p.dropless:
            if p.drop_mode == DROP_FULLSEQUENCE:
                _, dec = gather_full_sequence_decision(ctx, self.g.seq, dec, self.seq_len, E, p,
                                                      slots=self._fullseq_slots(ctx, T),
                                                      status=self.status, want_global=False)
            else:
                dec.kept = kept_mask(dec, T, E, p).bool()
        kept_in = None if p.dropless else dec.kept.to(torch.uint8).contiguous()
        seg = 0
        if self.pad_to_capacity and not p.dropless and p.drop_mode != DROP_FULLSEQUENCE:
            cap = capacity_limit(p.capacity_factor, T, E)
            seg = (cap + ALIGN - 1) // ALIGN * ALIGN
            plan = K.dispatch_plan(dec.experts, dec.gates, E, cap=cap, kept_in=kept_in, align=-seg)
        else:
            plan = K.dispatch_plan(dec.experts, dec.gates, E, cap=0, kept_in=kept_in)
        self.seg = seg
        self.align = -seg if seg else ALIGN
        saved = {"x": x, "dec": dec, "plan_dev": plan, "logits": logits}
        if self.single:
            self._mark_status()
            # padded expert-major layout straight from the plan; group sizes stay on device
            if seg:
                R = E * seg
            else:
                R = T * k + E * (ALIGN - 1)
                R = (R + ALIGN - 1) // ALIGN * ALIGN
            xp = K.permute(x, plan.gemm_row, R, poffsets=plan.poffsets, counts=plan.counts, E=E,
                           align=self.align)
            goff = plan.poffsets
            pre, h, y = X.ffn_forward(xp, goff, E, None, self.pk, R)
            ys = self._shared_forward(x, saved)
            out = K.combine(y, plan.gemm_row, T, gates=dec.gates, out=ys, accumulate=ys is not None)
            saved.update(xp=xp, pre=pre, h=h, y=y, goff=goff, G=E, gexp=None, R=R,
                         pair_row=plan.gemm_row)
            self._finish_forward(ctx, saved, plan.counts)
            return out, saved
        if not self.use_peer:
            self._mark_status()  # the NCCL path also checks it with its count all-gather
        out, saved = self._forward_exchange(ctx, x, dec, plan, saved)
        if "xpl" in saved:
            recv = saved["xpl"].recv_counts
        else:
            px = saved["peer"]
            te, ep_idx = px.te, px.me // px.etp
            recv = px.counts().view(px.members, E)[te::px.etp, ep_idx * self.L:(ep_idx + 1) * self.L].clone()
        self._finish_forward(ctx, saved, recv)
        return out, saved

    # ---- the reference-facing DispatchPlan and the wire ledger.  The layer's
    # exchanges are charged to a SimWorld ledger in the reference's call order
    # (dispatcher.py:309-361 forward, 425-468 backward): EP all_to_all_v,
    # exchange_meta, [ETP all_gather_v, exchange_meta, reduce_scatter_v], EP
    # all_to_all_v back; the counts stay on the device until the ledger is read.
    def _finish_forward(self, ctx, saved, recv):
        plan, dec = saved["plan_dev"], saved["dec"]
        ep = len(self.g.ep)
        saved["plan"] = DispatchPlan(plan, dec.n_tokens, self.k, ep, self.L, pair_gates=dec.gates,
                                     recv_src=recv)
        self._account(ctx, saved["plan"], meta=True)

    def _account(self, ctx, dplan: "DispatchPlan", meta: bool):
        if ctx is None or getattr(ctx.world, "account", None) is None:
            return
        H, ep, L_ = self.pk.hidden, dplan.ep_size, dplan.local_experts
        cnt = dplan.dev.counts
        ctx.account(self.g.ep, "all_to_all_v", H, lambda: cnt.view(ep, L_).sum(1))
        if meta:
            ctx.account(self.g.ep, None)
        if len(self.g.etp) > 1:
            ctx.account(self.g.etp, "all_gather_v", H, lambda: dplan.recv_counts.sum())
            if meta:
                ctx.account(self.g.etp, None)
            ctx.account(self.g.etp, "reduce_scatter_v", H, lambda: dplan.recv_counts.sum())
        ctx.account(self.g.ep, "all_to_all_v", H, lambda: dplan.recv_counts.sum(1))

    def _fullseq_slots(self, ctx, T: int) -> int:
        """Tokens per member of the full-sequence gather: the sequence group's
        largest block, agreed once (like the peer buffers); a later, larger
        block needs ``peer_tokens`` on first use."""
        cache = ctx.world.__dict__.setdefault("_fullseq_slots", {})
        key = (ctx.rank, self.g.seq)
        if key not in cache:
            mine = max(T, int(self.peer_tokens or 0))
            cache[key] = max(int(v) for v in ctx.meta(self.g.seq, mine).values())
        return cache[key]

    # ------------------------------------------------------- EP / ETP exchange
    # Rows are permuted straight into the padded per-global-expert layout,
    # which is destination-major with every (dest, local expert) chunk padded
    # to ALIGN rows.  One all_to_all_single per direction then lands them as
    # (sender, local expert) segments that are already GEMM-aligned, so the
    # receive side needs no regroup copy and the return trip restores the
    # sender's layout exactly (combine reads it through gemm_row).
    def _exchange_plan(self, ctx, plan) -> ExchangePlan:
        g = self.g
        ep_pos = g.ep.index(self.rank)
        if self.seg:
            # pad-to-capacity: static sizes, no count exchange, no host sync
            counts = np.full((len(g.ep), self.E), self.seg, dtype=np.int64)
            etp_recv = None
            if len(g.etp) > 1:
                etp_recv = np.full((len(g.etp), len(g.ep) * self.L), self.seg, dtype=np.int64)
            return exchange_plan(counts, ep_pos, self.L, etp_recv, ALIGN)
        # [ep, E] host (one sync), with every member's step status appended
        got = ctx.gather_counts(g.ep, torch.cat([plan.counts.to(torch.int64), self.status.to(torch.int64)]))
        counts = got[:, :-1]
        bad = [int(v) for v in got[:, -1]]
        if any(bad):
            _raise_status(bad[ep_pos] or ST_PEER_ABORT)
        mine = exchange_plan(counts, ep_pos, self.L, None, ALIGN)
        if len(g.etp) > 1:
            etp_recv = ctx.gather_counts(g.etp, torch.as_tensor(mine.recv_padded.reshape(-1)))
            return exchange_plan(counts, ep_pos, self.L, etp_recv, ALIGN)
        return mine

    def _gather_blocks(self, ctx, xp: ExchangePlan, mine: torch.Tensor) -> torch.Tensor:
        g = self.g
        if len(g.etp) == 1:
            return mine
        off = xp.block_off
        full = torch.empty((int(off[-1]), mine.shape[1]), dtype=mine.dtype, device=mine.device)
        sends = [(r, mine) for r in g.etp]
        recvs = [(g.etp[m], full[off[m]:off[m + 1]]) for m in range(len(g.etp))]
        ctx.p2p(g.etp, sends, recvs)
        return full

    def _reduce_blocks(self, ctx, xp: ExchangePlan, full: torch.Tensor) -> torch.Tensor:
        g = self.g
        if len(g.etp) == 1:
            return full
        off = xp.block_off
        me = g.etp.index(self.rank)
        n_me = int(off[me + 1] - off[me])
        parts = [torch.empty((n_me, full.shape[1]), dtype=full.dtype, device=full.device)
                 for _ in g.etp]
        sends = [(g.etp[m], full[off[m]:off[m + 1]]) for m in range(len(g.etp))]
        recvs = [(g.etp[m], parts[m]) for m in range(len(g.etp))]
        ctx.p2p(g.etp, sends, recvs)
        acc = parts[0].float()
        for q in parts[1:]:  # ascending ETP rank (collectives.py:386-388)
            acc += q.float()
        return acc.to(full.dtype)

    # ---- overlapped EP exchange (ETP = 1): while NCCL moves the remote rows,
    # the rank's own rows (its self segment of the send buffer) run through
    # the FFN; the remote segments follow once they land.
    def _overlap_groups(self, xpl: ExchangePlan):
        me = self.g.ep.index(self.rank)
        L_ = self.L
        dev = self.device
        so_me = int(sum(xpl.send_splits[:me]))
        n_self = int(xpl.send_splits[me])
        self_pad = xpl.recv_padded[me]
        soff = np.concatenate(([0], np.cumsum(self_pad))).astype(np.int64)
        go, ge, gx = [], [], []
        for s in range(len(self.g.ep)):
            if s == me:
                continue
            for le in range(L_):
                i = s * L_ + le
                go.append(xpl.group_off[i])
                ge.append(xpl.group_off[i + 1])
                gx.append(le)
        go.append(xpl.group_off[-1])  # bound for the elementwise kernels
        pin = lambda v: torch.tensor(v, dtype=torch.int32).pin_memory().to(dev, non_blocking=True)  # noqa: E731
        return dict(me=me, so_me=so_me, n_self=n_self, s_off=pin(soff.tolist()), G_self=L_,
                    r_off=pin(go), r_end=pin(ge), r_exp=pin(gx), G_rem=len(gx))

    def _forward_overlap(self, ctx, x, dec, plan, saved):
        T, H = x.shape
        E = self.E
        xpl = self._exchange_plan(ctx, plan)
        R_send, R_recv = int(sum(xpl.send_splits)), int(sum(xpl.recv_splits))
        xs = K.permute(x, plan.gemm_row, max(R_send, 1), poffsets=plan.poffsets, counts=plan.counts, E=E,
                       align=self.align)
        xr = torch.empty((max(R_recv, 1), H), dtype=x.dtype, device=x.device)
        work = ctx.a2a_single(self.g.ep, xs, xpl.send_splits, xr, xpl.recv_splits, async_op=True)
        og = self._overlap_groups(xpl)
        s_pre = s_h = s_y = None
        if og["n_self"]:
            xs_self = xs[og["so_me"]:og["so_me"] + og["n_self"]]
            s_pre, s_h, s_y = X.ffn_forward(xs_self, og["s_off"], og["G_self"], None, self.pk,
                                            og["n_self"])
        work.wait()
        r_pre, r_h, r_y = X.ffn_forward(xr, og["r_off"], og["G_rem"], og["r_exp"], self.pk, R_recv,
                                        gend=og["r_end"])
        ys = torch.empty((max(R_send, 1), H), dtype=x.dtype, device=x.device)
        work = ctx.a2a_single(self.g.ep, r_y, xpl.recv_splits, ys, xpl.send_splits, async_op=True)
        y_sh = self._shared_forward(x, saved)  # overlaps the return transfer
        work.wait()
        if s_y is not None:  # self rows never left the GPU
            ys[og["so_me"]:og["so_me"] + og["n_self"]].copy_(s_y)
        out = K.combine(ys, plan.gemm_row, T, gates=dec.gates, out=y_sh, accumulate=y_sh is not None)
        saved.update(xs=xs, xr=xr, s_pre=s_pre, s_h=s_h, r_pre=r_pre, r_h=r_h, y=ys, og=og, xpl=xpl,
                     pair_row=plan.gemm_row, R_send=R_send, R_recv=R_recv, overlap=True)
        return out, saved

    def _backward_overlap(self, ctx, u, sv, dec, plan):
        H = u.shape[1]
        E = self.E
        xpl, og = sv["xpl"], sv["og"]
        dys, dgates = K.permute_bwd(u, sv["pair_row"], dec.gates, sv["y"], poffsets=plan.poffsets,
                                    counts=plan.counts, E=E, align=self.align)
        dyr = torch.empty((max(sv["R_recv"], 1), H), dtype=u.dtype, device=u.device)
        work = ctx.a2a_single(self.g.ep, dys, xpl.send_splits, dyr, xpl.recv_splits, async_op=True)
        a, n = og["so_me"], og["n_self"]
        s_dx = None
        if n:
            s_dx, s_dw1, s_dw2 = X.ffn_backward(dys[a:a + n], sv["xs"][a:a + n], sv["s_pre"],
                                                sv["s_h"], og["s_off"], og["G_self"], None, self.pk, n)
        work.wait()
        r_dx, r_dw1, r_dw2 = X.ffn_backward(dyr, sv["xr"], sv["r_pre"], sv["r_h"], og["r_off"],
                                            og["G_rem"], og["r_exp"], self.pk, sv["R_recv"],
                                            gend=og["r_end"])
        rows = torch.empty((max(sv["R_send"], 1), H), dtype=u.dtype, device=u.device)
        work = ctx.a2a_single(self.g.ep, r_dx, xpl.recv_splits, rows, xpl.send_splits, async_op=True)
        # per-expert weight grads: self groups are experts 0..L-1, remote groups cycle le
        dw1p = r_dw1.reshape(-1, self.L, *r_dw1.shape[1:]).sum(0)
        dw2p = r_dw2.reshape(-1, self.L, *r_dw2.shape[1:]).sum(0)
        if s_dx is not None:
            dw1p += s_dw1
            dw2p += s_dw2
        work.wait()
        if s_dx is not None:
            rows[a:a + n].copy_(s_dx)
        return rows, dgates, dw1p, dw2p

    # ---- device-side EP exchange over NVLink peer memory (peer.py).  Tokens
    # are pushed straight from the token block into the owners' receive
    # buffers (no send buffer, no host sync), the GEMMs run on the receive
    # buffer with one group per local expert, and the second GEMM's epilogue
    # stores every output row straight back into the padded layout of the
    # rank it came from, so the combines read local memory.
    def _peer(self, ctx, T: int):
        from . import peer as PX

        H = self.pk.hidden
        cache = ctx.world.__dict__.setdefault("_peer_exchanges", {})
        xch = self.g.xch
        key = (ctx.rank, xch, self.E, self.k, H, self.peer_tag)
        px = cache.get(key)
        if px is None:
            # buffer layout must be identical on every member: agree on the
            # largest token block and on the push mode once, when the buffers
            # are created.  Deduplicated push: it trades link bytes for a local
            # copy of the duplicate rows; measured worth it from top-4 up (C4:
            # 1-2 % of the step), neutral or slightly worse at top-2
            env = os.environ.get("B200MOE_PUSH_DEDUP")
            dedup = env == "1" or (env is None and self.k >= 4)
            got = ctx.meta(xch, (max(int(self.peer_tokens or 0), T), dedup))
            T_max = max(int(v[0]) for v in got.values())
            if len({bool(v[1]) for v in got.values()}) != 1:
                raise ProtocolError("B200MOE_PUSH_DEDUP differs between the members of the exchange "
                                    f"{xch}: {[bool(got[r][1]) for r in xch]}")
            cap = PX.capacity_rows(len(xch), T_max, self.k, self.L, ALIGN, self.peer_capacity)
            ret = T_max * self.k + self.E * (ALIGN - 1)  # this rank's padded pair layout
            if self.pad_to_capacity and not self.params.dropless:
                seg = (capacity_limit(self.params.capacity_factor, T_max, self.E) + ALIGN - 1) // ALIGN
                ret = max(ret, self.E * seg * ALIGN)
            ret = (ret + ALIGN - 1) // ALIGN * ALIGN
            px = PX.PeerExchange(ctx, xch, self.E, self.L, H, cap, ret, self.device, etp=len(self.g.etp),
                                 dedup=dedup)
            px.tokens = T_max
            cache[key] = px
        return px

    def _forward_peer(self, ctx, x, dec, plan, saved):
        T = x.shape[0]
        px = self._peer(ctx, T)
        oversize = T > px.tokens
        ov = self.push_overlap and _overlap_fits(ctx)
        if oversize:
            # the block does not fit the peers' buffers: take part in the
            # step's protocol without tokens and fail it everywhere (status)
            self.status.bitwise_or_(ST_OVERSIZE)
            st = px.forward_dispatch(x[:0], dec.experts[:0], plan, ALIGN, status=self.status, overlap=ov)
        else:
            st = px.forward_dispatch(x, dec.experts, plan, ALIGN, status=self.status, overlap=ov)
        self._mark_status()
        if ov:
            # the NVLink push runs on the exchange stream beside GEMM1 over
            # this rank's own rows; GEMM1 over the received rows follows the
            # landing barrier (pre / h identical to one launch)
            pre, h = X.ffn_forward_split(px.region("xr"), st["goff"], self.L, self.pk, px.cap, st["split"],
                                         lambda: px.land(st), px.scatter("yret"))
        else:
            pre, h, _ = X.ffn_forward(px.region("xr"), st["goff"], self.L, None, self.pk, px.cap,
                                      y_scatter=px.scatter("yret"))
        y_sh, sh_done = self._shared_forward_side(x, saved)
        px.barrier()  # every expert output row (ETP: every partial) is back in yret
        if sh_done is not None:
            torch.cuda.current_stream().wait_event(sh_done)
        if oversize:
            out = torch.zeros_like(x)
            saved.update(peer=px, pst=st, pre=pre, h=h, pair_row=plan.gemm_row, y=None)
            return out, saved
        if px.etp == 1:
            y = px.region("yret")[0]
            out = K.combine(y, plan.gemm_row, T, gates=dec.gates, out=y_sh, accumulate=y_sh is not None)
        else:
            # ETP: the members' partial rows are folded inside the combine,
            # which also keeps the reduced rows (y_perm) for the backward
            y = torch.empty((px.ret_rows, px.H), dtype=x.dtype, device=x.device)
            out = K.combine(px.region("yret"), plan.gemm_row, T, gates=dec.gates, out=y_sh,
                            accumulate=y_sh is not None, rows_out=y)
        saved.update(peer=px, pst=st, pre=pre, h=h, pair_row=plan.gemm_row, y=y)
        return out, saved

    def _backward_peer(self, ctx, u, sv, dec, plan):
        px, st = sv["peer"], sv["pst"]
        px.check_generation(st)
        ov = self.push_overlap and "split" in st
        dgates = px.backward_dispatch(u, dec.experts, plan, dec.gates, st, sv["y"], ALIGN, status=self.status,
                                      overlap=ov)
        _, dw1p, dw2p = X.ffn_backward(px.region("dyr"), px.region("xr"), sv["pre"], sv["h"],
                                       st["goff"], self.L, None, self.pk, px.cap,
                                       dx_scatter=px.scatter("dxret"),
                                       split=st["split"] if ov else None, land=lambda: px.land(st))
        sv["shared_side"] = self._shared_backward_side(u, sv)
        px.barrier()  # every input-gradient row (ETP: every partial) is back in dxret
        # ETP: the partial rows [etp, rows, H] are folded by the combine
        rows = px.region("dxret")[0] if px.etp == 1 else px.region("dxret")
        return rows, dgates, dw1p, dw2p

    def _forward_exchange(self, ctx, x, dec, plan, saved):
        T, H = x.shape
        E = self.E
        if self.use_peer:
            return self._forward_peer(ctx, x, dec, plan, saved)
        if len(self.g.etp) == 1 and self.overlap:
            return self._forward_overlap(ctx, x, dec, plan, saved)
        xpl = self._exchange_plan(ctx, plan)
        R_send = int(sum(xpl.send_splits))
        xs = K.permute(x, plan.gemm_row, max(R_send, 1), poffsets=plan.poffsets, counts=plan.counts, E=E,
                       align=self.align)
        R_recv = int(sum(xpl.recv_splits))
        xr = torch.empty((max(R_recv, 1), H), dtype=x.dtype, device=x.device)
        ctx.a2a_single(self.g.ep, xs, xpl.send_splits, xr, xpl.recv_splits)
        xp = self._gather_blocks(ctx, xpl, xr[:R_recv])
        # pinned + non_blocking: a pageable H2D copy would stall the host on the stream
        goff = torch.tensor(xpl.group_off, dtype=torch.int32).pin_memory().to(self.device, non_blocking=True)
        gexp = torch.tensor(xpl.group_expert, dtype=torch.int32).pin_memory().to(self.device, non_blocking=True)
        G = len(xpl.group_expert)
        R = xp.shape[0]
        pre, h, y = X.ffn_forward(xp, goff, G, gexp, self.pk, R)
        y_mine = self._reduce_blocks(ctx, xpl, y)
        ys = torch.empty((max(R_send, 1), H), dtype=x.dtype, device=x.device)
        ctx.a2a_single(self.g.ep, y_mine, xpl.recv_splits, ys, xpl.send_splits)
        y_sh = self._shared_forward(x, saved)
        out = K.combine(ys, plan.gemm_row, T, gates=dec.gates, out=y_sh, accumulate=y_sh is not None)
        saved.update(xp=xp, pre=pre, h=h, y=ys, goff=goff, G=G, gexp=gexp, R=R, xpl=xpl,
                     pair_row=plan.gemm_row, R_send=R_send, R_recv=R_recv)
        return out, saved

    # ---------------------------------------------------------------- bwd
    def backward(self, ctx, u: torch.Tensor, sv: dict):
        p = self.params
        x, dec, plan = sv["x"], sv["dec"], sv["plan_dev"]
        T, H = x.shape
        u = u.to(self.device, self.dtype).contiguous()
        if tuple(u.shape) != tuple(x.shape):
            raise ValidationError(f"upstream shape {tuple(u.shape)} does not match input {tuple(x.shape)}",
                                  constraint="upstream-shape")
        self._account(ctx, sv["plan"], meta=False)
        E = self.E
        if self.single:
            dyp, dgates = K.permute_bwd(u, sv["pair_row"], dec.gates, sv["y"], poffsets=plan.poffsets,
                                        counts=plan.counts, E=E, align=self.align)
            dxp, dw1g, dw2g = X.ffn_backward(dyp, sv["xp"], sv["pre"], sv["h"], sv["goff"], sv["G"],
                                            None, self.pk, sv["R"])
            dw1p, dw2p = dw1g, dw2g
            rows = dxp
        elif sv.get("peer") is not None:
            rows, dgates, dw1p, dw2p = self._backward_peer(ctx, u, sv, dec, plan)
        elif sv.get("overlap"):
            rows, dgates, dw1p, dw2p = self._backward_overlap(ctx, u, sv, dec, plan)
        else:
            xpl = sv["xpl"]
            dys, dgates = K.permute_bwd(u, sv["pair_row"], dec.gates, sv["y"], poffsets=plan.poffsets,
                                        counts=plan.counts, E=E, align=self.align)
            dyr = torch.empty((max(sv["R_recv"], 1), H), dtype=u.dtype, device=u.device)
            ctx.a2a_single(self.g.ep, dys, xpl.send_splits, dyr, xpl.recv_splits)
            dyp = self._gather_blocks(ctx, xpl, dyr[:sv["R_recv"]])
            dxp, dw1g, dw2g = X.ffn_backward(dyp, sv["xp"], sv["pre"], sv["h"], sv["goff"], sv["G"],
                                            sv["gexp"], self.pk, sv["R"])
            # groups (member, sender, le) -> local experts, summed in group order
            dw1p = dw1g.reshape(-1, self.L, *dw1g.shape[1:]).sum(0)
            dw2p = dw2g.reshape(-1, self.L, *dw2g.shape[1:]).sum(0)
            dx_mine = self._reduce_blocks(ctx, xpl, dxp)
            rows = torch.empty((max(sv["R_send"], 1), H), dtype=u.dtype, device=u.device)
            ctx.a2a_single(self.g.ep, dx_mine, xpl.recv_splits, rows, xpl.send_splits)
        wg_tc = self.wg_parts is not None and K.router_wgrad_tc_supported(x, E)
        dz = K.router_bwd(dgates, dec.scores, dec.experts, dec.gates, GATE_CODES[p.gate_fn],
                          p.renormalize_topk, want_parts=wg_tc)
        if wg_tc:
            dz, dz_parts = dz
        side = sv.pop("shared_side", None)
        if side is not None:
            dx_sh, sv["shared_grads"], done = side
            torch.cuda.current_stream().wait_event(done)
        else:
            dx_sh, sv["shared_grads"] = self._shared_backward(u, sv)
        if E <= 8:
            # router term dz . W_g^T fused into the combine (W_g^T slice held in
            # registers, csrc/dispatch.cu combine_router_kernel for bf16)
            dx = K.combine(rows, sv["pair_row"], T, gates=None, dz=dz, w_gT=self.wgT, out=dx_sh,
                           accumulate=dx_sh is not None)
        else:
            dx = K.combine(rows, sv["pair_row"], T, gates=None, out=dx_sh, accumulate=dx_sh is not None)
            K.router_term(dz, self.wg, dx, parts=self.wg_parts)
        # dW_g = x^T dz: x read once by TMA, tensor cores against the exact
        # bf16 parts of dz written by router_bwd (router_tc.cu)
        if wg_tc:
            dwg = K.router_wgrad_tc(x, dz_parts, E)
        else:
            dwg = K.router_wgrad(x, dz, tc=self.wg_parts is not None)
        return dx, dwg, dw1p, dw2p


# ============================================================ layer API
def exchange_group(topology: ParallelTopology, rank: int) -> Tuple[int, ...]:
    """The EP x ETP block of ``rank``: EP and ETP are the innermost MoE axes
    in both layouts, so it is ep*etp consecutive ranks, ordered ep-major."""
    te, e, _, _ = topology.moe_coords(rank)
    base = rank - (e * topology.etp + te)
    return tuple(base + i for i in range(topology.ep * topology.etp))


def exchange_groups(topology: ParallelTopology) -> List[Tuple[int, ...]]:
    return sorted({exchange_group(topology, r) for r in range(topology.world_size)})


def _rank_groups(topology, groups: GroupSets, rank: int) -> LayerGroups:
    return LayerGroups(groups.group_of("moe", "EP", rank), groups.group_of("moe", "ETP", rank),
                       groups.group_of("moe", "EDP", rank), tuple(range(topology.world_size)),
                       sequence_group(topology, rank), exchange_group(topology, rank))


def _validate(blocks, topology, params, seq_len):
    if topology.pp != 1:
        raise ValidationError("numeric execution requires pp == 1", constraint="pp==1")
    if len(blocks) != topology.world_size:
        raise ValidationError(f"{len(blocks)} blocks for world_size {topology.world_size}",
                              constraint="blocks==world")
    groups = generate_parallel_groups(topology)
    verdict = check_pp_consistency(groups)
    if not verdict.consistent:
        raise ValidationError(f"pipeline groups differ between meshes: {verdict.mismatch}",
                              constraint="pp-consistency")
    E = params.num_experts
    if E % topology.ep or topology.ep > E:
        raise ValidationError(f"ep={topology.ep} must divide num_experts={E}", constraint="ep|E")
    if (not params.dropless) and params.drop_mode == DROP_FULLSEQUENCE and seq_len is None:
        raise ValidationError("full-sequence dropping needs seq_len", constraint="seq_len-required")
    return groups


def moe_forward(blocks, weights_map, topology: ParallelTopology, params: GatingParams, world,
                seq_len: Optional[int] = None, workers: Optional[int] = None, *, dtype=None,
                check_finite_inputs: bool = True, shared_weights: Optional[X.ExpertWeights] = None,
                pad_to_capacity: bool = False, exchange: Optional[str] = None,
                peer_tokens: Optional[int] = None, peer_tag=0, peer_capacity: Optional[float] = None):
    """Run the MoE layer forward on every rank of ``world`` (dispatcher.py:246-384).

    ``world`` is a LocalWorld (all ranks in this process) or an NcclWorld
    (this process's rank only; other entries of the returned list are None).
    ``dtype`` selects the compute precision (torch.float32 parity mode or
    torch.bfloat16); default: the dtype of the blocks' values (fp64 -> fp32).
    ``exchange`` picks the EP all-to-all: "peer" (device-side over NVLink
    peer memory; bf16) or "nccl"; default $B200MOE_EP_EXCHANGE or "peer".
    The peer buffers are allocated on first use for the largest token block
    of that call (or ``peer_tokens`` if larger); layers whose forward and
    backward interleave need distinct ``peer_tag`` values (their own buffers).
    The receive buffers hold the worst case (every sender's tokens routed to
    one rank) unless ``peer_capacity`` = f sizes them for f times the
    balanced load; a step whose routing overflows them then raises
    ``ProtocolError`` on every rank (no rank traps).
    """
    pending = world.__dict__.pop("_b200moe_pending", None)
    if pending is not None:  # a previous step whose backward never ran
        _check_step(pending, block=True)
    groups = _validate(blocks, topology, params, seq_len)
    if hasattr(world, "setup_groups"):
        world.setup_groups([groups.moe["EP"], groups.moe["ETP"], groups.moe["EDP"],
                            [tuple(range(topology.world_size))],
                            sorted({sequence_group(topology, r) for r in range(topology.world_size)}),
                            exchange_groups(topology)])

    def program(ctx):
        rank = ctx.rank
        b = blocks[rank]
        etp_idx, ep_idx, _, _ = topology.moe_coords(rank)
        w = weights_map[(ep_idx, etp_idx)]
        dev = world.device_of(rank) if hasattr(world, "device_of") else getattr(world, "device", torch.device("cuda"))
        dt = dtype or (b.values.dtype if b.values.dtype in (torch.float32, torch.bfloat16) else torch.float32)
        layer = RankLayer(params, w, topology, _rank_groups(topology, groups, rank), rank, dt, dev,
                          seq_len, check=check_finite_inputs, shared=shared_weights,
                          pad_to_capacity=pad_to_capacity, exchange=exchange,
                          peer_tokens=max([int(peer_tokens or 0)] + [b_.values.shape[0] for b_ in blocks
                                                                     if b_ is not None]),
                          peer_tag=peer_tag, peer_capacity=peer_capacity)
        out, saved = layer.forward(ctx, b.values, b.positions)
        saved["layer"] = layer
        return out, saved

    results = world.run(program, workers=workers)
    context = ForwardContext(world, topology, params, weights_map, groups)
    outputs = []
    for r in results:
        outputs.append(None if r is None else r[0])
        context.per_rank.append(None if r is None else r[1])
    for sv in context.per_rank:
        if sv is not None:
            sv["decision"] = sv["dec"]
    # failures the device flagged during the step (non-finite inputs, an
    # oversized block, a failed peer, duplicate positions) are raised here if
    # the step's status copy has already landed, otherwise at the next
    # natural synchronisation point -- the start of moe_backward for this
    # context, or the next moe_forward on this world -- so the host never
    # stalls the stream it feeds
    if not _check_step(context, block=False):
        world.__dict__["_b200moe_pending"] = context
    return outputs, context


def _check_step(context: ForwardContext, block: bool) -> bool:
    """Raise the root cause of a step the device flagged; False when
    ``block`` is off and a status copy is still in flight."""
    if context.__dict__.get("_checked"):
        return True
    layers = [(r, sv["layer"]) for r, sv in enumerate(context.per_rank) if sv is not None]
    events = [layer.status_event for _, layer in layers if layer.status_event is not None]
    if not block and not all(ev.query() for ev in events):
        return False
    for ev in events:
        ev.synchronize()
    context.__dict__["_checked"] = True
    bits = {r: int(layer.status_host[0]) if layer.status_event is not None else 0 for r, layer in layers}
    for mask in (ST_NONFINITE, ST_DUPLICATE, ST_OVERSIZE, ST_RECV_OVERFLOW, ST_PEER_ABORT):  # root cause first
        for r in sorted(bits):
            if bits[r] & mask:
                if mask == ST_NONFINITE:
                    raise nonfinite_error(context.per_rank[r]["x"], context.params, f" (rank {r})")
                _raise_status(mask, f" (rank {r})")
    return True


def moe_backward(upstream, context: ForwardContext, workers: Optional[int] = None) -> BackwardResult:
    """Gradients of sum over ranks of <upstream, output> (dispatcher.py:387-510)."""
    topology = context.topology
    # the forward's status, if it has landed (it normally has); a flagged step
    # pushes nothing in the backward either (the exchange kernels check the
    # same word), so an unchecked status is raised after the backward or by
    # the next moe_forward -- never a host stall in a pipelined loop
    if _check_step(context, block=False) and context.world.__dict__.get("_b200moe_pending") is context:
        del context.world.__dict__["_b200moe_pending"]
    if len(upstream) != topology.world_size:
        raise ValidationError(f"{len(upstream)} upstream blocks for world_size {topology.world_size}",
                              constraint="upstream==world")
    world_group = tuple(range(topology.world_size))

    def program(ctx):
        sv = context.per_rank[ctx.rank]
        layer: RankLayer = sv["layer"]
        u = upstream[ctx.rank]
        if not isinstance(u, torch.Tensor):
            u = torch.as_tensor(np.asarray(u, dtype=np.float64))
        dx, dwg, dw1p, dw2p = layer.backward(ctx, u, sv)
        if topology.world_size > 1:
            dwg = ctx.all_reduce(world_group, dwg, "sum")
        else:  # the reference all-reduces over a world of one too (a zero-byte ledger record)
            ctx.account(world_group, "all_reduce", 1, dwg.numel())
        if len(layer.g.edp) > 1:
            flat = torch.cat([dw1p.reshape(-1), dw2p.reshape(-1)])
            red = ctx.all_reduce(layer.g.edp, flat, "sum")
            dw1p = red[: dw1p.numel()].reshape(dw1p.shape)
            dw2p = red[dw1p.numel():].reshape(dw2p.shape)
        shared = None
        if sv.get("shared_grads") is not None:
            s1, s2 = sv["shared_grads"]
            if topology.world_size > 1:  # replicated shared expert: data-parallel over all ranks
                flat = ctx.all_reduce(world_group, torch.cat([s1.reshape(-1), s2.reshape(-1)]), "sum")
                s1, s2 = flat[: s1.numel()].reshape(s1.shape), flat[s1.numel():].reshape(s2.shape)
            shared = (X.unpack_w1_grad(s1, layer.shared_pk.act)[0], X.unpack_w2_grad(s2)[0])
        return dx, dwg, dw1p, dw2p, layer.pk.act, shared

    results = context.world.run(program, workers=workers)
    if _check_step(context, block=False) and context.world.__dict__.get("_b200moe_pending") is context:
        del context.world.__dict__["_b200moe_pending"]
    elif not context.__dict__.get("_checked"):
        context.world.__dict__["_b200moe_pending"] = context
    input_grads = [None if r is None else r[0] for r in results]
    w_g_grad = next(r[1] for r in results if r is not None)
    shared = next(r[5] for r in results if r is not None)
    expert_grads = {}
    for rank, r in enumerate(results):
        if r is None:
            continue
        etp_idx, ep_idx, edp_idx, _ = topology.moe_coords(rank)
        if edp_idx == 0:
            expert_grads[(ep_idx, etp_idx)] = (X.unpack_w1_grad(r[2], r[4]), X.unpack_w2_grad(r[3]))
    return BackwardResult(input_grads, w_g_grad, expert_grads, shared)
