"""Folded parallel meshes (host-side only): attention TP x CP x DP x PP and MoE
ETP x EP x EDP x PP over the same ranks.

Mirrors /root/reference/pkg/src/moefold/topology.py (ParallelTopology
:41-122, GroupSets :125-144, generate_parallel_groups :191-215,
check_pp_consistency :218-234, sequence_group :248-256).  On the B200 path
these groups become NCCL communicators; nothing here touches the GPU.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

from .errors import ValidationError

LAYOUT_PP_OUTERMOST = "pp-outermost"
LAYOUT_LISTING1 = "listing1"
LAYOUTS = (LAYOUT_PP_OUTERMOST, LAYOUT_LISTING1)

Group = Tuple[int, ...]


@dataclass(frozen=True)
class ParallelTopology:
    world_size: int
    tp: int = 1
    cp: int = 1
    pp: int = 1
    ep: int = 1
    etp: int = 1
    layout: str = LAYOUT_PP_OUTERMOST

    def __post_init__(self):
        if self.world_size < 1:
            raise ValidationError(f"world_size must be >= 1, got {self.world_size}",
                                  constraint="world_size>=1")
        for name in ("tp", "cp", "pp", "ep", "etp"):
            deg = getattr(self, name)
            if deg < 1:
                raise ValidationError(f"{name} must be >= 1, got {deg}", constraint=f"{name}>=1")
            if self.world_size % deg:
                raise ValidationError(f"{name}={deg} does not divide world_size={self.world_size}",
                                      constraint=f"{name}|world_size")
        for label, prod in (("tp*cp*pp", self.tp * self.cp * self.pp),
                            ("etp*ep*pp", self.etp * self.ep * self.pp)):
            if self.world_size % prod:
                raise ValidationError(f"{label}={prod} does not divide world_size={self.world_size}",
                                      constraint=f"{label}|world_size")
        if self.layout not in LAYOUTS:
            raise ValidationError(f"layout must be one of {LAYOUTS}, got {self.layout!r}",
                                  constraint="layout")

    @property
    def dp(self) -> int:
        return self.world_size // (self.tp * self.cp * self.pp)

    @property
    def edp(self) -> int:
        return self.world_size // (self.etp * self.ep * self.pp)

    # axis order (slowest first) of each mesh, with degrees
    def _attn_axes(self):
        if self.layout == LAYOUT_LISTING1:
            return (("DP", self.dp), ("PP", self.pp), ("CP", self.cp), ("TP", self.tp))
        return (("PP", self.pp), ("DP", self.dp), ("CP", self.cp), ("TP", self.tp))

    def _moe_axes(self):
        if self.layout == LAYOUT_LISTING1:
            return (("EDP", self.edp), ("PP", self.pp), ("EP", self.ep), ("ETP", self.etp))
        return (("PP", self.pp), ("EDP", self.edp), ("EP", self.ep), ("ETP", self.etp))

    @staticmethod
    def _decompose(rank: int, axes) -> Dict[str, int]:
        coords = {}
        for name, deg in reversed(axes):
            coords[name] = rank % deg
            rank //= deg
        return coords

    def attn_coords(self, rank: int) -> Tuple[int, int, int, int]:
        """(tp, cp, dp, pp) of ``rank`` -- topology.py:100-110."""
        c = self._decompose(rank, self._attn_axes())
        return c["TP"], c["CP"], c["DP"], c["PP"]

    def moe_coords(self, rank: int) -> Tuple[int, int, int, int]:
        """(etp, ep, edp, pp) of ``rank`` -- topology.py:112-122."""
        c = self._decompose(rank, self._moe_axes())
        return c["ETP"], c["EP"], c["EDP"], c["PP"]


@dataclass(frozen=True)
class GroupSets:
    attention: Dict[str, List[Group]]
    moe: Dict[str, List[Group]]

    def group_of(self, mesh: str, dim: str, rank: int) -> Group:
        table = self.attention if mesh == "attention" else self.moe
        for g in table[dim]:
            if rank in g:
                return g
        raise ValidationError(f"rank {rank} not found in any {mesh}/{dim} group",
                              constraint="rank-in-group")


def _groups_along(axes, dim: str) -> List[Group]:
    """Rank groups varying ``dim`` with the other axes fixed, enumerated in
    row-major order of the remaining axes."""
    names = [n for n, _ in axes]
    degs = dict(axes)
    strides = {}
    s = 1
    for name, deg in reversed(axes):
        strides[name] = s
        s *= deg
    others = [n for n in names if n != dim]
    out = []
    for combo in itertools.product(*[range(degs[n]) for n in others]):
        base = sum(c * strides[n] for n, c in zip(others, combo))
        out.append(tuple(base + i * strides[dim] for i in range(degs[dim])))
    return out


def generate_parallel_groups(topology: ParallelTopology) -> GroupSets:
    """Rank groups of both meshes -- topology.py:191-215."""
    a_axes, m_axes = topology._attn_axes(), topology._moe_axes()
    attention = {n: _groups_along(a_axes, n) for n, _ in a_axes}
    moe = {n: _groups_along(m_axes, n) for n, _ in m_axes}
    return GroupSets(attention=attention, moe=moe)


@dataclass(frozen=True)
class PpConsistency:
    consistent: bool
    mismatch: Optional[Tuple[Group, Group]] = None


def check_pp_consistency(groups: GroupSets) -> PpConsistency:
    """Both meshes must induce the same pipeline groups -- topology.py:218-234."""
    moe_sets = {frozenset(g) for g in groups.moe["PP"]}
    owner = {r: g for g in groups.moe["PP"] for r in g}
    for g in groups.attention["PP"]:
        if frozenset(g) not in moe_sets:
            return PpConsistency(False, (g, owner[min(g)]))
    return PpConsistency(True, None)


def sequence_group(topology: ParallelTopology, rank: int) -> Group:
    """Ranks holding shards of ``rank``'s sequences (its TP x CP block) --
    topology.py:248-256."""
    _, _, d, p = topology.attn_coords(rank)
    return tuple(r for r in range(topology.world_size)
                 if topology.attn_coords(r)[2:] == (d, p))


SPAN_INTRA = "intra"
SPAN_INTER = "inter"


@dataclass(frozen=True)
class ClusterModel:
    """Node size for span classification of rank groups (topology.py:148-165).
    Defaults describe one 8 x B200 NVLink-5 / NVSwitch node: 900 GB/s per
    GPU per direction inside the node."""

    node_size: int = 8
    intra_bw: float = 900e9
    inter_bw: float = 50e9
    per_link_latency_s: float = 5e-6
    peak_flops: float = 2250e12

    def __post_init__(self):
        if self.node_size < 1:
            raise ValidationError("node_size must be >= 1", constraint="node_size>=1")
        if self.intra_bw <= 0 or self.inter_bw <= 0:
            raise ValidationError("bandwidths must be > 0", constraint="bw>0")
        if self.inter_bw > self.intra_bw:
            raise ValidationError("inter_bw must not exceed intra_bw", constraint="inter_bw<=intra_bw")


@dataclass(frozen=True)
class GroupSpan:
    span: str  # SPAN_INTRA or SPAN_INTER
    node_count: int


def classify_group_span(group: Group, cluster: ClusterModel) -> GroupSpan:
    """Whether a rank group fits in one node; ranks fill nodes in contiguous
    blocks of node_size (topology.py:237-245)."""
    if len(group) == 0:
        raise ValidationError("cannot classify an empty group", constraint="group-nonempty")
    nodes = {r // cluster.node_size for r in group}
    return GroupSpan(SPAN_INTRA if len(nodes) == 1 else SPAN_INTER, len(nodes))
