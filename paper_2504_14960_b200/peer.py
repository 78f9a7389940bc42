"""EP all-to-all over NVLink peer memory (replaces dispatcher.py:310-361 and
430-466 of the reference for ETP = 1).

Every member of an EP group maps one symmetric buffer:

    [flags | count matrix | xr | yr | dyr | dxr]

``xr`` receives the token rows routed to this rank's experts (pushed by the
senders' dispatch kernels straight from their token blocks), ``yr`` holds the
expert outputs the senders pull back in their combine kernels; ``dyr`` /
``dxr`` are the backward twins.  Split sizes never reach the host: every
sender writes its per-expert counts into row ``me`` of every peer's count
matrix and each rank derives all receive layouts on the device.

On an NcclWorld the buffer comes from torch symmetric memory (one mapping per
peer over NVLink) and ranks synchronise with a flag barrier kernel.  On a
LocalWorld (ranks as threads on one GPU) each rank owns an ordinary device
buffer, the addresses are exchanged with exchange_meta and the barrier is a
host rendezvous after a stream synchronize -- the same kernels run on both.
"""
from __future__ import annotations

from typing import Dict, Tuple

import torch

from . import kernels as K
from .collectives import LocalRankContext, NcclRankContext
from .errors import ProtocolError

_FLAG_BYTES = 4096
_REGION_ALIGN = 1 << 16
REGIONS = ("xr", "yr", "dyr", "dxr")


def _up(n: int, a: int) -> int:
    return (n + a - 1) // a * a


def capacity_rows(ep: int, T_max: int, k: int, L_: int, align: int) -> int:
    """Receive rows a rank can need: every sender routes each of its tokens
    to at most min(k, L) of this rank's experts, plus one pad per expert."""
    return ep * T_max * min(k, L_) + L_ * (align - 1)


class PeerExchange:
    """Symmetric buffers + device exchange of one EP group, as seen by one rank."""

    def __init__(self, ctx, group: Tuple[int, ...], E: int, L_: int, H: int, cap_rows: int, device):
        self.group = tuple(group)
        self.ep = len(group)
        self.me = self.group.index(ctx.rank)
        self.E, self.L, self.H, self.cap = E, L_, H, int(cap_rows)
        self.ctx = ctx
        self.device = device
        self.cnt_off = _FLAG_BYTES
        off = _up(self.cnt_off + self.ep * E * 4, _REGION_ALIGN)
        self.off: Dict[str, int] = {}
        region = _up(self.cap * H * 2, _REGION_ALIGN)
        for r in REGIONS:
            self.off[r] = off
            off += region
        self.nbytes = off
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
        got = ctx.exchange_meta(self.group, self.buf.data_ptr())
        self.peer_base = torch.tensor([int(got[r]) for r in self.group], dtype=torch.int64,
                                      device=self.device)
        torch.cuda.current_stream().synchronize()
        self.device_barrier = False

    def region(self, name: str) -> torch.Tensor:
        """This rank's [cap, H] bf16 view of a region."""
        o = self.off[name]
        n = self.cap * self.H * 2
        return self.buf[o:o + n].view(torch.bfloat16).view(self.cap, self.H)

    def counts(self) -> torch.Tensor:
        """This rank's copy of the [ep, E] count matrix."""
        return self.buf[self.cnt_off:self.cnt_off + self.ep * self.E * 4].view(torch.int32)

    # ------------------------------------------------------------ sync
    def barrier(self):
        """All members' prior stream work (local and remote writes) is visible."""
        if self.device_barrier:
            self.epoch += 1
            K.ep_barrier(self.peer_base, 0, self.me, self.ep, self.epoch)
        else:
            torch.cuda.current_stream().synchronize()
            self.ctx.exchange_meta(self.group, None)

    # ------------------------------------------------------------ steps
    def forward_dispatch(self, x, topk_idx, plan, align: int):
        """counts push -> barrier -> layout -> pad zero -> dispatch -> barrier.
        Returns the saved routing state (seg_off, goff, gcount, pair_dst, pair_rrow)."""
        K.ep_counts_push(plan.counts, self.me, self.ep, self.peer_base, self.cnt_off)
        self.barrier()
        seg_off, goff, gcount = K.ep_layout(self.counts(), self.me, self.ep, self.L, align, self.cap)
        K.ep_zero_pads(self.region("xr"), goff, gcount, self.L, align)
        pd, pr = K.ep_dispatch(x, topk_idx, plan.gemm_row, plan.poffsets, seg_off, self.L,
                               self.peer_base, self.off["xr"])
        self.barrier()
        self.generation += 1
        return dict(seg_off=seg_off, goff=goff, gcount=gcount, pair_dst=pd, pair_rrow=pr,
                    generation=self.generation)

    def check_generation(self, st):
        if st["generation"] != self.generation:
            raise ProtocolError("peer receive buffers were reused by another forward before this "
                                "backward: give interleaved layers distinct peer tags")
