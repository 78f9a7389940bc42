"""Rank worlds and the variable-count collectives of the MoE layer.

Mirrors the reference's per-rank API (/root/reference/pkg/src/moefold/
collectives.py: VarBuffer :42-78, SimWorld.run :128-173, RankContext
.all_to_all_v / all_gather_v / reduce_scatter_v / all_reduce / exchange_meta
:260-327) with device tensors instead of numpy arrays.

Two worlds implement it:
  * ``NcclWorld``  -- production: one process per GPU (torchrun), collectives
    over NCCL process groups built from the folded EP/ETP/EDP meshes.
  * ``LocalWorld`` -- N ranks as threads of one process, like SimWorld: all on
    one GPU (the parity tests run multi-rank topologies on a single B200) or
    one GPU each (``devices=[...]``: the in-process multi-GPU shim, peer
    access enabled between the devices).  Collectives are device copies
    performed by the last rank to arrive.  No kernel ever waits on another
    rank's kernel, so the ranks cannot deadlock the GPUs.

``SimWorld`` is a LocalWorld that also keeps the reference's wire ledger
(TrafficRecord per collective, collectives.py:81-92, 104-126): the layer's
implicit exchanges (the peer push, the scatter epilogue, NCCL) are charged
exactly as the reference's all_to_all_v / all_gather_v / reduce_scatter_v /
all_reduce would charge them, from the device-resident plan counts, which are
read only when the ledger is inspected.  ``traffic_stats`` aggregates it by
primitive and node span (collectives.py:452-466).

Both also provide the engine-level primitives ``p2p`` (a batch of row-chunk
sends/receives), ``meta`` (exchange_meta that is not part of the reference
call sequence) and ``gather_counts`` (all-gather of small int vectors to host
memory).
"""
from __future__ import annotations

import threading
from dataclasses import dataclass, field
from typing import Any, Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from .errors import ProtocolError, ValidationError
from .topology import ClusterModel, classify_group_span

Group = Tuple[int, ...]
_STALL_TIMEOUT_S = 120.0


@dataclass
class VarBuffer:
    """Variable-count row payload: ``values`` [sum(counts), row_width]."""

    values: torch.Tensor
    row_width: int
    counts: np.ndarray

    def __post_init__(self):
        self.counts = np.asarray(self.counts, dtype=np.int64).ravel()
        if self.row_width < 1:
            raise ValidationError("row_width must be >= 1", constraint="row_width>=1")
        if np.any(self.counts < 0):
            raise ValidationError("counts must be >= 0", constraint="counts>=0")
        if self.values.numel() != self.row_width * int(self.counts.sum()):
            raise ValidationError(
                f"values length {self.values.numel()} != row_width {self.row_width} * total rows "
                f"{int(self.counts.sum())}", constraint="values==row_width*sum(counts)")
        self.values = self.values.reshape(-1, self.row_width)

    @classmethod
    def from_rows(cls, rows: torch.Tensor, counts=None) -> "VarBuffer":
        if rows.dim() != 2:
            raise ValidationError("from_rows expects a 2-D tensor", constraint="rows-2d")
        return cls(rows, rows.shape[1], [rows.shape[0]] if counts is None else counts)

    def rows(self) -> torch.Tensor:
        return self.values


def _check_group(rank: int, group: Group):
    if rank not in group:
        raise ProtocolError(f"rank {rank} called a collective on group {group} it is not part of")
    if any(group[i] >= group[i + 1] for i in range(len(group) - 1)):
        raise ProtocolError(f"group must list distinct ranks in ascending order, got {group}")


# =============================================================== LocalWorld
class _Slot:
    __slots__ = ("payloads", "results", "remaining")

    def __init__(self):
        self.payloads: Dict[int, Any] = {}
        self.results: Optional[Dict[int, Any]] = None
        self.remaining = 0


class LocalWorld:
    """N ranks as threads of one process (SimWorld analogue), on one device
    or -- with ``devices`` -- one device per rank.

    ``device_barrier``: every rank issues its work on its own CUDA stream and
    the peer exchange synchronises ranks with the device-side flag barrier
    (ep_barrier_kernel) instead of a host rendezvous -- the production
    (NcclWorld) synchronisation path, runnable on a single GPU.  Host-side
    collectives then synchronise the ranks' streams around every exchange."""

    def __init__(self, n_ranks: int, device=None, devices: Optional[Sequence] = None,
                 device_barrier: bool = False):
        if n_ranks < 1:
            raise ValidationError("n_ranks must be >= 1", constraint="n_ranks>=1")
        self.n_ranks = n_ranks
        dev = torch.device(device or "cuda")
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.devices = None
        if devices is not None:
            if len(devices) != n_ranks:
                raise ValidationError(f"{len(devices)} devices for {n_ranks} ranks",
                                      constraint="devices==ranks")
            self.devices = [torch.device("cuda", torch.device(d).index if not isinstance(d, int) else d)
                            for d in devices]
            self.device = self.devices[0]
            _enable_peer_access(self.devices)
        self._cond = threading.Condition()
        self._slots: Dict[tuple, _Slot] = {}
        self._seq: Dict[tuple, int] = {}
        self._epoch = 0
        self._failure: Optional[BaseException] = None
        self.device_barrier = bool(device_barrier)
        self._streams = None
        if self.device_barrier and self.device.type == "cuda":
            self._streams = [torch.cuda.Stream(device=self.device_of(r)) for r in range(n_ranks)]

    def run(self, program: Callable[["RankContext"], Any], *, workers: Optional[int] = None) -> List[Any]:
        with self._cond:
            self._epoch += 1
            self._failure = None
            self._seq = {}
            self._slots = {}
        results: List[Any] = [None] * self.n_ranks
        errors: Dict[int, BaseException] = {}

        def runner(rank: int):
            try:
                if self.device_of(rank).type == "cuda":
                    torch.cuda.set_device(self.device_of(rank))
                if self._streams is not None:
                    s = self._streams[rank]
                    s.wait_stream(torch.cuda.current_stream())  # inputs made on the caller's stream
                    with torch.cuda.stream(s):
                        results[rank] = program(LocalRankContext(self, rank))
                    torch.cuda.current_stream().wait_stream(s)
                else:
                    results[rank] = program(LocalRankContext(self, rank))
            except _Aborted:
                pass
            except BaseException as exc:  # noqa: BLE001
                errors[rank] = exc
                with self._cond:
                    if self._failure is None:
                        self._failure = exc
                    self._cond.notify_all()

        if self.n_ranks == 1:
            runner(0)
        else:
            threads = [threading.Thread(target=runner, args=(r,), daemon=True) for r in range(self.n_ranks)]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
        if self._failure is not None:
            raise self._failure
        if errors:
            raise errors[min(errors)]
        return results

    def device_of(self, rank: int) -> torch.device:
        return self.devices[rank] if self.devices is not None else self.device

    def _rendezvous(self, rank: int, group: Group, payload: Any,
                    compute: Callable[[Group, Dict[int, Any]], Dict[int, Any]]) -> Any:
        _check_group(rank, group)
        if self._streams is not None:
            # ranks run on their own streams: a payload (or a device result
            # computed by the last arrival) is complete before it crosses over
            torch.cuda.current_stream().synchronize()
        with self._cond:
            if self._failure is not None:
                raise _Aborted()
            key = (group, rank)
            seq = self._seq.get(key, 0)
            self._seq[key] = seq + 1
            skey = (self._epoch, seq, group)
            slot = self._slots.setdefault(skey, _Slot())
            slot.payloads[rank] = payload
            if len(slot.payloads) == len(group):
                slot.results = compute(group, slot.payloads)
                if self._streams is not None:
                    torch.cuda.current_stream().synchronize()
                slot.remaining = len(group)
                slot.payloads = {}
                self._cond.notify_all()
            else:
                while slot.results is None and self._failure is None:
                    if not self._cond.wait(timeout=_STALL_TIMEOUT_S):
                        exc = ProtocolError(
                            f"collective rendezvous stalled: group {group} waited for "
                            f"{sorted(set(group) - set(slot.payloads))} (round {seq})")
                        self._failure = exc
                        self._cond.notify_all()
                        raise exc
            if self._failure is not None:
                raise _Aborted()
            out = slot.results[rank]
            slot.remaining -= 1
            if slot.remaining == 0:
                del self._slots[skey]
        return out


@dataclass(frozen=True)
class TrafficRecord:
    """One collective's wire elements per member, group order (collectives.py:81-92)."""

    epoch: int
    seq: int
    group: Group
    primitive: str
    row_width: int
    elements_sent: Tuple[int, ...]

    @property
    def total_elements(self) -> int:
        return int(sum(self.elements_sent))


def _host(v):
    if callable(v):
        v = v()
    if isinstance(v, torch.Tensor):
        v = v.detach().cpu().numpy()
    return np.asarray(v, dtype=np.int64)


def _wire(primitive: str, group: Group, width: int, pay: Dict[int, Any]) -> Tuple[int, ...]:
    """Elements each member puts on the wire, by the reference's rules
    (collectives.py:341-417): self traffic is free, all_gather_v charges
    own_rows * (n-1), reduce_scatter_v total - own partition, all_reduce the
    ring 2(n-1)/n of the buffer."""
    n = len(group)
    vals = [_host(pay[r]) for r in group]
    if primitive == "all_to_all_v":
        return tuple(int((v.sum() - v[i]) * width) for i, v in enumerate(vals))
    if primitive == "all_gather_v":
        return tuple(int(v.sum()) * (n - 1) * width for v in vals)
    if primitive == "reduce_scatter_v":
        total = sum(int(v.sum()) for v in vals)
        return tuple((total - int(v.sum())) * width for v in vals)
    if primitive == "all_reduce":
        return tuple(int(round(int(v.sum()) * 2 * (n - 1) / n)) if n > 1 else 0 for v in vals)
    raise ValidationError(f"unknown primitive {primitive!r}", constraint="primitive")


class SimWorld(LocalWorld):
    """LocalWorld plus the reference's traffic ledger (collectives.py:104-126).

    Every rank deposits its share of each collective through ``account`` in
    the reference's call order; a deposit is an int, a host array, a device
    tensor or a callable returning one, resolved only when ``ledger`` is read
    (so the layer never synchronises for the accounting).  ``run`` may be
    called repeatedly (forward, then backward); the ledger accumulates."""

    def __init__(self, n_ranks: int, device=None, devices: Optional[Sequence] = None):
        super().__init__(n_ranks, device=device, devices=devices)
        self._acct_lock = threading.Lock()
        self._acct: Dict[tuple, list] = {}
        self._acct_seq: Dict[tuple, int] = {}

    def account(self, rank: int, group: Group, primitive: Optional[str], width: int = 1,
                payload: Any = 0) -> None:
        """Rank ``rank``'s contribution to its next collective on ``group``;
        ``primitive`` None stands for an exchange_meta (it takes a sequence
        number, like the reference's rendezvous, but is not wire-accounted)."""
        group = tuple(group)
        _check_group(rank, group)
        with self._acct_lock:
            key = (self._epoch, group, rank)
            seq = self._acct_seq.get(key, 0)
            self._acct_seq[key] = seq + 1
            if primitive is None:
                return
            slot = self._acct.setdefault((self._epoch, seq, group), [primitive, int(width), {}])
            if slot[0] != primitive:
                raise ProtocolError(f"{primitive}: rank {rank} disagrees with {slot[0]} on group {group} "
                                    f"(round {seq})")
            slot[2][rank] = payload

    @property
    def ledger(self) -> List[TrafficRecord]:
        """Traffic records in a deterministic order (round, then group)."""
        out = []
        with self._acct_lock:
            items = sorted(self._acct.items())
        for (epoch, seq, group), (prim, width, pay) in items:
            if len(pay) != len(group):
                raise ProtocolError(f"{prim} on {group} (round {seq}): ranks "
                                    f"{sorted(set(group) - set(pay))} never contributed")
            out.append(TrafficRecord(epoch, seq, group, prim, width, _wire(prim, group, width, pay)))
        return out


@dataclass
class TrafficStats:
    """Ledger bytes aggregated by primitive and span (collectives.py:440-450)."""

    by_primitive_span: Dict[Tuple[str, str], float] = field(default_factory=dict)

    def bytes_for(self, primitive: str, span: Optional[str] = None) -> float:
        if span is not None:
            return self.by_primitive_span.get((primitive, span), 0.0)
        return sum(v for (p, _), v in self.by_primitive_span.items() if p == primitive)

    @property
    def total_bytes(self) -> float:
        return sum(self.by_primitive_span.values())


def traffic_stats(world: SimWorld, cluster: Optional[ClusterModel] = None,
                  elem_bytes: float = 8.0) -> TrafficStats:
    """Per-primitive, per-span byte totals of ``world``'s ledger
    (collectives.py:452-466); ``elem_bytes`` converts elements to bytes
    (2 for the bf16 rows the B200 path actually moves)."""
    cluster = cluster or ClusterModel()
    stats = TrafficStats()
    for rec in world.ledger:
        key = (rec.primitive, classify_group_span(rec.group, cluster).span)
        stats.by_primitive_span[key] = stats.by_primitive_span.get(key, 0.0) + rec.total_elements * elem_bytes
    return stats


def _enable_peer_access(devices) -> None:
    """Let kernels on every device dereference the others' memory (the peer
    exchange stores into peer buffers directly)."""
    from . import _lib as L

    lib = L.load()
    cur = torch.cuda.current_device()
    try:
        for a in devices:
            torch.cuda.set_device(a)
            for b in devices:
                if a != b:
                    L.check(lib.b200moe_enable_peer_access(b.index), "b200moe_enable_peer_access")
    finally:
        torch.cuda.set_device(cur)


class _Aborted(BaseException):
    pass


class _Done:
    """Handle of an already-completed (emulated) collective."""

    def wait(self):
        return None


class _Work:
    """Handle of an in-flight NCCL collective; wait() makes the current
    stream wait for it (no host synchronisation)."""

    def __init__(self, work, prof=None):
        self.work = work
        self.prof = prof

    def wait(self):
        self.work.wait()
        if self.prof is not None:
            from . import _lib

            _lib.PROFILE.end(*self.prof)


class RankContext:
    """Per-rank handle (collectives.py:249-327 analogue)."""

    rank: int
    n_ranks: int

    # reference-API collectives -------------------------------------------
    def all_to_all_v(self, group: Group, send: VarBuffer) -> VarBuffer:
        if len(send.counts) != len(group):
            raise ProtocolError(f"all_to_all_v: rank {self.rank} supplied {len(send.counts)} counts "
                                f"for a group of {len(group)}")
        w = send.row_width
        self.account(group, "all_to_all_v", w, send.counts.copy())
        all_counts = self.gather_counts(group, torch.as_tensor(send.counts, dtype=torch.int64))
        me = group.index(self.rank)
        recv_counts = all_counts[:, me]
        out = torch.empty((int(recv_counts.sum()), w), dtype=send.values.dtype, device=send.values.device)
        so = np.concatenate(([0], np.cumsum(send.counts)))
        ro = np.concatenate(([0], np.cumsum(recv_counts)))
        sends = [(group[j], send.values[so[j]:so[j + 1]]) for j in range(len(group))]
        recvs = [(group[j], out[ro[j]:ro[j + 1]]) for j in range(len(group))]
        self.p2p(group, sends, recvs)
        return VarBuffer(out, w, recv_counts)

    def all_gather_v(self, group: Group, send: VarBuffer) -> Tuple[VarBuffer, np.ndarray]:
        if len(send.counts) != 1:
            raise ProtocolError(f"all_gather_v: rank {self.rank} must supply a single row count")
        w = send.row_width
        self.account(group, "all_gather_v", w, int(send.counts[0]))
        counts = self.gather_counts(group, torch.as_tensor(send.counts, dtype=torch.int64))[:, 0]
        out = torch.empty((int(counts.sum()), w), dtype=send.values.dtype, device=send.values.device)
        off = np.concatenate(([0], np.cumsum(counts)))
        sends = [(r, send.values) for r in group]
        recvs = [(group[j], out[off[j]:off[j + 1]]) for j in range(len(group))]
        self.p2p(group, sends, recvs)
        return VarBuffer(out, w, counts), counts

    def reduce_scatter_v(self, group: Group, values: torch.Tensor, partition_counts: Sequence[int],
                         row_width: int) -> torch.Tensor:
        counts = np.asarray(partition_counts, dtype=np.int64)
        if len(counts) != len(group):
            raise ProtocolError(f"reduce_scatter_v: rank {self.rank} supplied {len(counts)} "
                                f"partitions for a group of {len(group)}")
        vals = values.reshape(-1, row_width)
        if vals.shape[0] != int(counts.sum()):
            raise ProtocolError(f"reduce_scatter_v: rank {self.rank} buffer rows {vals.shape[0]} != "
                                f"partition total {int(counts.sum())}")
        off = np.concatenate(([0], np.cumsum(counts)))
        me = group.index(self.rank)
        mine = counts[me]
        self.account(group, "reduce_scatter_v", row_width, int(mine))
        parts = [torch.empty((int(mine), row_width), dtype=vals.dtype, device=vals.device)
                 for _ in group]
        sends = [(group[j], vals[off[j]:off[j + 1]]) for j in range(len(group))]
        recvs = [(group[j], parts[j]) for j in range(len(group))]
        self.p2p(group, sends, recvs)
        total = parts[0].clone()
        for p in parts[1:]:  # fold in ascending rank order (collectives.py:386-388)
            total += p
        return total

    def all_reduce(self, group: Group, values: torch.Tensor, op: str = "sum") -> torch.Tensor:
        if op not in ("sum", "avg"):
            raise ValidationError(f"all_reduce op must be sum or avg, got {op!r}", constraint="op")
        self.account(group, "all_reduce", 1, int(values.numel()))
        return self._all_reduce(group, values, op)

    def exchange_meta(self, group: Group, payload: Any) -> Dict[int, Any]:
        """All-gather of host objects (collectives.py:420-423); on a SimWorld
        it takes a ledger sequence number like the reference's rendezvous."""
        self.account(group, None)
        return self.meta(group, payload)

    def meta(self, group: Group, payload: Any) -> Dict[int, Any]:
        """exchange_meta for the engine's own bookkeeping (buffer agreement,
        host barriers): not part of the reference's call sequence."""
        raise NotImplementedError

    def account(self, group: Group, primitive: Optional[str], width: int = 1, payload: Any = 0) -> None:
        """Charge this rank's share of a collective to the world's ledger
        (SimWorld only; a no-op elsewhere).  See SimWorld.account."""
        acct = getattr(self.world, "account", None)
        if acct is not None:
            acct(self.rank, group, primitive, width, payload)

    # engine primitives ---------------------------------------------------
    def p2p(self, group: Group, sends: List[Tuple[int, torch.Tensor]],
            recvs: List[Tuple[int, torch.Tensor]]) -> None:
        raise NotImplementedError

    def all_gather_fixed(self, group: Group, t: torch.Tensor) -> torch.Tensor:
        """[len(group), *t.shape]: every member's equally-shaped tensor in
        group order, on this rank's device -- no sizes cross the host, so the
        stream never waits for the host (NCCL all_gather_into_tensor)."""
        raise NotImplementedError

    def a2a_single(self, group: Group, send: torch.Tensor, send_splits: Sequence[int],
                   recv: torch.Tensor, recv_splits: Sequence[int], async_op: bool = False):
        """Rows [sum(send_splits[:j]), +send_splits[j]) of ``send`` go to
        member j; ``recv`` receives members' rows in ascending member order.
        With async_op the call returns a handle whose wait() orders the
        current stream after the transfer (emulated worlds complete eagerly)."""
        so = np.concatenate(([0], np.cumsum(send_splits))).astype(np.int64)
        ro = np.concatenate(([0], np.cumsum(recv_splits))).astype(np.int64)
        sends = [(group[j], send[so[j]:so[j + 1]]) for j in range(len(group))]
        recvs = [(group[j], recv[ro[j]:ro[j + 1]]) for j in range(len(group))]
        self.p2p(group, sends, recvs)
        return _Done() if async_op else None

    def gather_counts(self, group: Group, counts: torch.Tensor) -> np.ndarray:
        """[len(group), n] int64 on the host: row i = member i's vector."""
        raise NotImplementedError

    def _all_reduce(self, group, values, op):
        raise NotImplementedError


class LocalRankContext(RankContext):
    def __init__(self, world: LocalWorld, rank: int):
        self.world = world
        self.rank = rank
        self.n_ranks = world.n_ranks

    def meta(self, group, payload):
        return self.world._rendezvous(self.rank, group, payload,
                                      lambda g, p: {r: dict(p) for r in g})

    def gather_counts(self, group, counts):
        host = counts.detach().to("cpu", torch.int64).numpy().copy()
        got = self.meta(group, host)
        return np.stack([np.asarray(got[r]).ravel() for r in group])

    def p2p(self, group, sends, recvs):
        payload = (list(sends), list(recvs))

        def compute(g, payloads):
            # i-th send A->B pairs with the i-th recv on B from A (NCCL order)
            for b in g:
                seen: Dict[int, int] = {}
                for src, dst in payloads[b][1]:
                    i = seen.get(src, 0)
                    seen[src] = i + 1
                    mine = [t for (peer, t) in payloads[src][0] if peer == b]
                    if i >= len(mine):
                        raise ProtocolError(f"p2p: rank {b} expects a message from {src} that was not sent")
                    t = mine[i]
                    if t.numel() != dst.numel():
                        raise ProtocolError(f"p2p: size mismatch {src}->{b}: {t.numel()} vs {dst.numel()}")
                    if t.numel():
                        dst.copy_(t.reshape(dst.shape))
            return {r: None for r in g}

        self.world._rendezvous(self.rank, group, payload, compute)

    def all_gather_fixed(self, group, t):
        def compute(g, payloads):
            shapes = {tuple(payloads[r].shape) for r in g}
            if len(shapes) != 1:
                raise ProtocolError(f"all_gather_fixed: shapes differ across the group: {shapes}")
            return {r: torch.stack([payloads[q].to(payloads[r].device) for q in g]) for r in g}

        return self.world._rendezvous(self.rank, group, t.contiguous(), compute)

    def _all_reduce(self, group, values, op):
        def compute(g, payloads):
            total = payloads[g[0]].clone()
            for r in g[1:]:
                total += payloads[r].to(total.device)
            if op == "avg":
                total /= len(g)
            return {r: total.to(payloads[r].device, copy=True) for r in g}

        return self.world._rendezvous(self.rank, group, values, compute)


# ================================================================ NcclWorld
class NcclWorld:
    """One process per GPU over torch.distributed (NCCL on B200, gloo on CPU
    for host-logic tests).  Call ``setup_groups`` with every group list the
    layer will use, identically on all ranks, before the first collective."""

    def __init__(self):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise ValidationError("torch.distributed is not initialised", constraint="dist-init")
        self.dist = dist
        self.n_ranks = dist.get_world_size()
        self.rank = dist.get_rank()
        self._pgs: Dict[Group, Any] = {}
        self.device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")

    def setup_groups(self, group_lists: Sequence[Sequence[Group]]) -> None:
        for glist in group_lists:
            for g in glist:
                g = tuple(g)
                if g in self._pgs:
                    continue
                if len(g) == self.n_ranks:
                    self._pgs[g] = None  # default group
                else:
                    self._pgs[g] = self.dist.new_group(list(g))

    def pg(self, group: Group):
        if group not in self._pgs:
            if len(group) == self.n_ranks:
                return None
            raise ProtocolError(f"process group {group} was not set up (call setup_groups)")
        return self._pgs[group]

    def run(self, program, *, workers=None) -> List[Any]:
        out: List[Any] = [None] * self.n_ranks
        out[self.rank] = program(NcclRankContext(self))
        return out


class NcclRankContext(RankContext):
    def __init__(self, world: NcclWorld):
        self.world = world
        self.rank = world.rank
        self.n_ranks = world.n_ranks

    def meta(self, group, payload):
        _check_group(self.rank, group)
        objs: List[Any] = [None] * len(group)
        self.world.dist.all_gather_object(objs, payload, group=self.world.pg(group))
        return {r: o for r, o in zip(group, objs)}

    def gather_counts(self, group, counts):
        _check_group(self.rank, group)
        from . import _lib

        dev = self.world.device
        e0 = _lib.PROFILE.begin() if _lib.PROFILE.on else None
        c = counts.to(dev, torch.int64).reshape(-1).contiguous()
        out = torch.empty((len(group) * c.numel(),), dtype=torch.int64, device=dev)
        self.world.dist.all_gather_into_tensor(out, c, group=self.world.pg(group))
        host = out.cpu().numpy().reshape(len(group), c.numel())
        if e0 is not None:
            _lib.PROFILE.end("nccl:count_allgather+sync", e0)
        return host

    def p2p(self, group, sends, recvs):
        _check_group(self.rank, group)
        dist = self.world.dist
        pg = self.world.pg(group)
        ops = []
        self_sends = [t for (p, t) in sends if p == self.rank]
        self_recvs = [t for (p, t) in recvs if p == self.rank]
        if len(self_sends) != len(self_recvs):
            raise ProtocolError("p2p: unmatched self send/recv")
        for s, r in zip(self_sends, self_recvs):
            if s.numel():
                r.copy_(s.reshape(r.shape))
        for p, t in sends:
            if p != self.rank and t.numel():
                ops.append(dist.P2POp(dist.isend, t.contiguous(), p, group=pg))
        for p, t in recvs:
            if p != self.rank and t.numel():
                ops.append(dist.P2POp(dist.irecv, t, p, group=pg))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def all_gather_fixed(self, group, t):
        _check_group(self.rank, group)
        t = t.contiguous()
        out = torch.empty((len(group),) + tuple(t.shape), dtype=t.dtype, device=t.device)
        if len(group) == 1:
            out[0].copy_(t)
        else:
            self.world.dist.all_gather_into_tensor(out.view(-1), t.view(-1), group=self.world.pg(group))
        return out

    def a2a_single(self, group, send, send_splits, recv, recv_splits, async_op=False):
        from . import _lib

        _check_group(self.rank, group)
        ns, nr = int(sum(send_splits)), int(sum(recv_splits))
        if len(group) == 1:
            if ns:
                recv[:nr].copy_(send[:ns])
            return _Done() if async_op else None
        e0 = _lib.PROFILE.begin() if _lib.PROFILE.on else None
        work = self.world.dist.all_to_all_single(
            recv[:nr], send[:ns], [int(v) for v in recv_splits], [int(v) for v in send_splits],
            group=self.world.pg(group), async_op=async_op)
        if async_op:
            # (profiled span = issue .. wait, i.e. including overlapped compute)
            return _Work(work, None if e0 is None else (f"nccl:a2a_async[{ns}->{nr} rows]", e0))
        if e0 is not None:
            _lib.PROFILE.end(f"nccl:a2a[{ns}->{nr} rows]", e0)
        return None

    def _all_reduce(self, group, values, op):
        _check_group(self.rank, group)
        t = values.clone()
        self.world.dist.all_reduce(t, group=self.world.pg(group))
        if op == "avg":
            t /= len(group)
        return t
