"""EP all-to-all (and the ETP all-gather / reduce-scatter) over NVLink peer
memory (replaces dispatcher.py:309-362 and 425-468 of the reference).

The exchange group is the EP x ETP block of ranks (member = ep_idx * etp +
etp_idx).  A token row routed to EP index d is pushed to all etp members of
d (the ETP all-gather folded into the dispatch); each member computes its
F-shard's partial output and returns it into its own block of the sender's
return region, where the sender sums the blocks (the reduce-scatter).
Every member maps one symmetric buffer:

    [flags | count matrix | xr | dyr | origin | yret | dxret]

Receive side (rows routed to this rank's experts, expert-major, senders
contiguous -- the reference's ``grp_order`` layout): ``xr`` gets the token
rows, pushed by the senders' dispatch kernels straight from their token
blocks; ``origin`` records for every row (sender, row in the sender's padded
layout); ``dyr`` gets the backward's g*u rows.  Return side (this rank's own
pairs, in its padded expert-major layout): ``yret`` / ``dxret`` receive the
expert outputs / input gradients that the owners' GEMM epilogues store
directly over NVLink (gemm_tc epilogue 5), so the return all-to-all overlaps
the GEMM tile by tile and the combines read local memory.

Split sizes never reach the host: every sender writes its per-expert counts
into row ``me`` of every peer's count matrix and each rank derives all
receive layouts on the device.  On an NcclWorld the buffer comes from torch
symmetric memory (one mapping per peer over NVLink) and ranks synchronise
with a flag barrier kernel.  On a LocalWorld (ranks as threads on one GPU)
each rank owns an ordinary device buffer, the addresses are exchanged with
ctx.meta and the barrier is a host rendezvous after a stream
synchronize -- the same kernels run on both.
"""
from __future__ import annotations

import math
from typing import Dict, Optional, Tuple

import numpy as np

import torch

from . import kernels as K
from .collectives import LocalRankContext, NcclRankContext
from .errors import ProtocolError

_FLAG_BYTES = 4096
_REGION_ALIGN = 1 << 16


def _up(n: int, a: int) -> int:
    return (n + a - 1) // a * a


def capacity_rows(ep: int, T_max: int, k: int, L_: int, align: int, factor: Optional[float] = None) -> int:
    """Receive rows a rank can need: every sender routes each of its tokens
    to at most min(k, L) of this rank's experts, plus one pad per expert.
    ``factor`` f sizes for f times the balanced load (T_max * k rows) instead,
    capped at that worst case; an overflowing step fails cleanly (status)."""
    worst = ep * T_max * min(k, L_)
    rows = worst if factor is None else min(worst, int(math.ceil(factor * T_max * k)))
    return rows + L_ * (align - 1)


def wire_rows(send_counts, topology) -> int:
    """Token rows the exchange moves between GPUs in one layer step (forward
    + backward), from every rank's kept rows per EP destination
    (``send_counts[r]`` [ep, L], DispatchPlan.send_counts).

    A pair routed from rank r to EP index j is pushed to the etp members of
    j -- all but r itself cross the wire -- and each member returns its
    partial the same way; the backward repeats both.  This equals the
    reference SimWorld ledger's all_to_all_v + all_gather_v +
    reduce_scatter_v token rows (collectives.py:11-18; the a2a charges
    off-rank rows, the ETP gather (etp-1) rows per received row and the
    reduce-scatter the non-owned partials), which tests/test_cpu_host.py
    checks against the golden ledger."""
    etp = topology.etp
    total = 0
    for r, sc in enumerate(send_counts):
        _, e_idx, _, _ = topology.moe_coords(r)
        sc = [int(v) for v in np.asarray(sc).sum(axis=1)]
        total += sum(c * (etp - (1 if j == e_idx else 0)) for j, c in enumerate(sc))
    return 4 * total


class PeerExchange:
    """Symmetric buffers + device exchange of one EP x ETP block, as seen by
    one rank.  ``group`` lists the members in order ep_idx * etp + etp_idx.

    cap_rows: receive rows (xr/dyr/origin); ret_rows: rows of this rank's own
    padded pair layout (yret/dxret hold one such block per ETP member: the
    members' partial outputs, reduced by the receiver)."""

    def __init__(self, ctx, group: Tuple[int, ...], E: int, L_: int, H: int, cap_rows: int,
                 ret_rows: int, device, etp: int = 1, dedup: bool = False):
        self.group = tuple(group)
        self.members = len(group)
        self.etp = etp
        self.ep = self.members // etp
        self.me = self.group.index(ctx.rank)
        self.te = self.me % etp
        self.E, self.L, self.H = E, L_, H
        self.cap, self.ret_rows = int(cap_rows), int(ret_rows)
        self.ctx = ctx
        self.device = device
        self.cnt_off = _FLAG_BYTES
        off = _up(self.cnt_off + self.members * E * 4, _REGION_ALIGN)
        self.off: Dict[str, int] = {}
        for name, nbytes in (("xr", self.cap * H * 2), ("dyr", self.cap * H * 2),
                             ("origin", self.cap * 8), ("dup", self.cap * 8),
                             ("yret", etp * self.ret_rows * H * 2),
                             ("dxret", etp * self.ret_rows * H * 2)):
            self.off[name] = off
            off += _up(nbytes, _REGION_ALIGN)
        self.nbytes = off
        # one push per (token, remote EP index): only when an EP index hosts
        # more than one expert can two pairs of a token share a destination
        self.dedup = bool(dedup) and L_ >= 2
        self.epoch = 0
        self.generation = 0  # forwards run on these buffers (checked by backward)
        self._handle = None
        if isinstance(ctx, NcclRankContext):
            self._init_symmetric(ctx)
        elif isinstance(ctx, LocalRankContext):
            self._init_local(ctx)
        else:
            raise ProtocolError(f"peer exchange needs a LocalWorld or NcclWorld context, got {type(ctx)}")

    # ------------------------------------------------------------ buffers
    def _init_symmetric(self, ctx):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as sm

        pg = ctx.world.pg(self.group) or dist.group.WORLD
        self.buf = sm.empty(self.nbytes, dtype=torch.uint8, device=self.device)
        self.buf[:self.cnt_off].zero_()
        self._handle = sm.rendezvous(self.buf, pg)
        ptrs = [int(p) for p in self._handle.buffer_ptrs]
        self.peer_base = torch.tensor(ptrs, dtype=torch.int64, device=self.device)
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=pg)  # flags zeroed everywhere before the first epoch
        self.device_barrier = True

    def _init_local(self, ctx):
        self.buf = torch.zeros((self.nbytes,), dtype=torch.uint8, device=self.device)
        torch.cuda.current_stream().synchronize()  # zeroed flags before any peer's first barrier
        got = ctx.meta(self.group, self.buf.data_ptr())
        self.peer_base = torch.tensor([int(got[r]) for r in self.group], dtype=torch.int64,
                                      device=self.device)
        torch.cuda.current_stream().synchronize()
        # LocalWorld(device_barrier=True): ranks on their own streams meet in
        # the flag barrier kernel, as across GPUs; otherwise a host rendezvous
        self.device_barrier = bool(getattr(ctx.world, "device_barrier", False))

    def region(self, name: str) -> torch.Tensor:
        """This rank's bf16 view of a row region: [cap, H] (receive side) or
        [etp, ret_rows, H] (return side, one block per ETP member)."""
        o = self.off[name]
        if name in ("yret", "dxret"):
            n = self.etp * self.ret_rows * self.H * 2
            return self.buf[o:o + n].view(torch.bfloat16).view(self.etp, self.ret_rows, self.H)
        return self.buf[o:o + self.cap * self.H * 2].view(torch.bfloat16).view(self.cap, self.H)

    def returned(self, name: str) -> torch.Tensor:
        """The returned rows [ret_rows, H]: the single block, or the ETP
        members' partial blocks summed (reduce-scatter fold order)."""
        parts = self.region(name)
        return parts[0] if self.etp == 1 else K.ep_reduce_parts(parts)

    def dup(self) -> torch.Tensor:
        o = self.off["dup"]
        return self.buf[o:o + self.cap * 8].view(torch.int32).view(self.cap, 2)

    def origin(self) -> torch.Tensor:
        o = self.off["origin"]
        return self.buf[o:o + self.cap * 8].view(torch.int32).view(self.cap, 2)

    def counts(self) -> torch.Tensor:
        """This rank's copy of the [members, E] count matrix."""
        return self.buf[self.cnt_off:self.cnt_off + self.members * self.E * 4].view(torch.int32)

    def scatter(self, region: str):
        """Scatter-epilogue target: (row origin table, peer bases, byte offset
        of this ETP member's block in the senders' return region)."""
        return (self.origin(), self.peer_base, self.off[region] + self.te * self.ret_rows * self.H * 2)

    # ------------------------------------------------------------ sync
    def barrier(self):
        """All members' prior stream work (local and remote writes) is visible."""
        if self.device_barrier:
            self.epoch += 1
            K.ep_barrier(self.peer_base, 0, self.me, self.members, self.epoch)
        else:
            torch.cuda.current_stream().synchronize()
            self.ctx.meta(self.group, None)

    # ------------------------------------------------------------ steps
    def forward_dispatch(self, x, topk_idx, plan, align: int, status=None, overlap: bool = False):
        """counts push -> barrier -> layout -> pads -> dispatch -> barrier.
        Returns the routing state the rest of the step needs.  ``status``
        (device int32[1]): a rank whose step already failed pushes an abort
        marker instead of its counts, every member then skips the pushes and
        flags the step (bit 1), so all of them finish the barriers and raise.

        ``overlap``: the push is split (b200moe_ep_dispatch_part): the rows
        this rank routes to itself are stored on the compute stream, the
        NVLink part runs on the exchange stream beside the caller's first
        GEMM over those own rows (``st["split"]``: the GEMM groups of both
        halves); the caller then calls :meth:`land` before the GEMM over the
        received rows."""
        K.ep_counts_push(plan.counts, self.me, self.members, self.peer_base, self.cnt_off, status=status)
        self.barrier()
        seg_off, goff, gcount = K.ep_layout(self.counts(), self.me, self.ep, self.etp, self.L, align,
                                            self.cap, status=status)
        K.ep_zero_pads(self.region("xr"), goff, gcount, self.L, align, origin=self.origin())
        dup_off = self.off["dup"] if self.dedup else -1
        args = (x, topk_idx, plan.gemm_row, plan.poffsets, seg_off, self.L, self.peer_base, self.me,
                self.etp, self.off["xr"], self.off["origin"])
        st = dict(seg_off=seg_off, goff=goff, gcount=gcount)
        if overlap:
            st["split"] = K.ep_split_groups(self.counts(), self.me, self.ep, self.etp, self.L, seg_off,
                                            goff, gcount)
            K.ep_dispatch(*args, dup_off=dup_off, status=status, part=1)
            self._on_side(lambda: K.ep_dispatch(*args, dup_off=dup_off, status=status, part=2))
            st["pending"] = ("fwd",)
        else:
            K.ep_dispatch(*args, dup_off=dup_off, status=status)
            self.barrier()
            if self.dedup:
                K.ep_expand(self.region("xr"), goff, gcount, self.L, self.dup(), 0)
        self.generation += 1
        st["generation"] = self.generation
        return st

    def backward_dispatch(self, u, topk_idx, plan, gates, st, y_rows, align: int, status=None,
                          overlap: bool = False):
        """pads -> push g*u rows (dgates from the returned y) -> barrier.
        Nothing is pushed when the forward's ``status`` flagged the step.
        ``overlap``: as forward_dispatch (the caller runs the first backward
        GEMM over its own rows, then :meth:`land`)."""
        K.ep_zero_pads(self.region("dyr"), st["goff"], st["gcount"], self.L, align)
        dup_off = self.off["dup"] if self.dedup else -1
        args = (u, topk_idx, plan.gemm_row, plan.poffsets, st["seg_off"], self.L, self.peer_base, self.me,
                self.etp, self.off["dyr"])
        kw = dict(bwd=True, y_rows=y_rows, gates=gates, dup_off=dup_off, status=status)
        if overlap:
            dg = K.ep_dispatch(*args, part=1, **kw)
            self._on_side(lambda: K.ep_dispatch(*args, part=2, dgates=dg, **kw))
            st["pending"] = ("bwd",)
            return dg
        dg = K.ep_dispatch(*args, **kw)
        self.barrier()
        if self.dedup:
            K.ep_expand(self.region("dyr"), st["goff"], st["gcount"], self.L, self.dup(), 1)
            K.ep_expand(self.region("dyr"), st["goff"], st["gcount"], self.L, self.dup(), 2)
        return dg

    # ------------------------------------------------------------ overlap
    def _on_side(self, fn):
        """Run ``fn``'s launches on the exchange stream after everything the
        compute stream has queued so far."""
        main = torch.cuda.current_stream(self.device)
        if getattr(self, "stream", None) is None:
            self.stream = torch.cuda.Stream(device=self.device)
        self.stream.wait_stream(main)
        with torch.cuda.stream(self.stream):
            fn()

    def land(self, st):
        """Finish an overlapped push: barrier (+ dedup expansion) on the
        exchange stream; the compute stream then waits for it, so every
        received row is in place for the next GEMM."""
        kind = st.pop("pending", None)
        if kind is None:
            return
        main = torch.cuda.current_stream(self.device)

        def finish():
            self.barrier()
            if self.dedup:
                if kind[0] == "fwd":
                    K.ep_expand(self.region("xr"), st["goff"], st["gcount"], self.L, self.dup(), 0)
                else:
                    K.ep_expand(self.region("dyr"), st["goff"], st["gcount"], self.L, self.dup(), 1)
                    K.ep_expand(self.region("dyr"), st["goff"], st["gcount"], self.L, self.dup(), 2)

        with torch.cuda.stream(self.stream):
            finish()
        main.wait_stream(self.stream)

    def check_generation(self, st):
        if st["generation"] != self.generation:
            raise ProtocolError("peer receive buffers were reused by another forward before this "
                                "backward: give interleaved layers distinct peer tags")
