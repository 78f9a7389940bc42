"""Expert feed-forward networks (reference: /root/reference/pkg/src/moefold/experts.py).

Public API mirrors the reference (ExpertWeights :40-63, full_expert_matrices
:66-75, init_gating_matrix :78-81, init_expert_weights :84-127,
expert_forward_shard :130-143, expert_backward_shard :146-172).

B200 layout.  Weights live on the device packed per rank as
  w1p [L, N1, H]  (N1 = F_shard for relu/gelu, 2*F_shard for SwiGLU)
  w2p [L, H, F_shard]
i.e. K-major for the forward GEMMs.  SwiGLU's gate/up columns are interleaved
in 64-row blocks [32 gate | 32 up] so one accumulator tile holds matching
gate/up pairs.  Token rows are expert-major and padded to GEMM_ALIGN rows per
group; the grouped GEMMs read the group offsets from device memory.
"""
from __future__ import annotations

import warnings

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib as L
from . import kernels as K
from .errors import ValidationError

ACT_RELU = "relu"
ACT_GELU = "gelu"
ACT_SWIGLU = "swiglu"
ACTIVATIONS = (ACT_RELU, ACT_GELU, ACT_SWIGLU)


# --------------------------------------------------------------- packing
def swiglu_interleave_cols(w1: torch.Tensor) -> torch.Tensor:
    """[H, 2F] = [gate | up]  ->  [2F, H] rows in 64-blocks [32 gate | 32 up]."""
    H, F2 = w1.shape
    F = F2 // 2
    if F % 32:
        raise ValidationError("swiglu needs ffn % 32 == 0 per shard", constraint="swiglu-ffn%32")
    g = w1[:, :F].T.reshape(F // 32, 32, H)
    u = w1[:, F:].T.reshape(F // 32, 32, H)
    return torch.stack([g, u], dim=1).reshape(F2, H)


@dataclass
class PackedExperts:
    w1p: torch.Tensor  # [L, N1, H]
    w2p: torch.Tensor  # [L, H, F]
    act: str
    hidden: int
    ffn: int  # F_shard

    @property
    def n1(self) -> int:
        return self.w1p.shape[1]

    @property
    def local(self) -> int:
        return self.w1p.shape[0]

    @property
    def dtype(self):
        return self.w1p.dtype


def pack_experts(w1: Sequence, w2: Sequence, act: str, dtype, device) -> PackedExperts:
    mats1, mats2 = [], []
    for a, b in zip(w1, w2):
        a = torch.as_tensor(a).to(device=device)
        b = torch.as_tensor(b).to(device=device)
        if act == ACT_SWIGLU:
            mats1.append(swiglu_interleave_cols(a))
        else:
            mats1.append(a.T)
        mats2.append(b.T)
    w1p = torch.stack(mats1).to(dtype).contiguous()
    w2p = torch.stack(mats2).to(dtype).contiguous()
    H = w1p.shape[2]
    F = w2p.shape[2]
    return PackedExperts(w1p, w2p, act, H, F)


def unpack_w1_grad(dw1p: torch.Tensor, act: str) -> List[torch.Tensor]:
    """[L, N1, H] device grads (SwiGLU rows already [gate | up], see
    ffn_backward) -> list of reference-layout [H, N1] views (no copy)."""
    return [g.T for g in dw1p]


def unpack_w2_grad(dw2p: torch.Tensor) -> List[torch.Tensor]:
    return [g.T for g in dw2p]


# --------------------------------------------------------------- reference API
@dataclass
class ExpertWeights:
    """One rank's shard of its local experts (experts.py:40-63).

    ``w1[i]`` [hidden, ffn/etp] (SwiGLU: [hidden, 2*ffn/etp] = [gate|up]) and
    ``w2[i]`` [ffn/etp, hidden] of local expert ``expert_ids[i]``; numpy
    arrays or tensors.  ``packed(dtype, device)`` caches the device layout.
    """

    expert_ids: Tuple[int, ...]
    w1: List
    w2: List
    activation: str
    etp_rank: int
    etp_size: int
    _packed: Dict = field(default_factory=dict, repr=False, compare=False)

    def local_index(self, expert_id: int) -> int:
        try:
            return tuple(self.expert_ids).index(expert_id)
        except ValueError:
            raise ValidationError(
                f"expert {expert_id} is not hosted here (local: {self.expert_ids})",
                constraint="expert-local") from None

    def packed(self, dtype=torch.bfloat16, device=None) -> PackedExperts:
        device = torch.device(device or "cuda")
        key = (dtype, str(device))
        if key not in self._packed:
            self._packed[key] = pack_experts(self.w1, self.w2, self.activation, dtype, device)
        return self._packed[key]


def full_expert_matrices(num_experts: int, hidden: int, ffn: int, seed: int):
    """Unsharded matrices U(+-1/sqrt(H)) from rng([seed, 1]) -- experts.py:66-75."""
    rng = np.random.default_rng([seed, 1])
    bound = 1.0 / np.sqrt(hidden)
    w1 = [rng.uniform(-bound, bound, size=(hidden, ffn)) for _ in range(num_experts)]
    w2 = [rng.uniform(-bound, bound, size=(ffn, hidden)) for _ in range(num_experts)]
    return w1, w2


def full_swiglu_matrices(num_experts: int, hidden: int, ffn: int, seed: int):
    """Builder-defined SwiGLU init (no reference): per expert gate, up, down
    U(+-1/sqrt(H)) from rng([seed, 4]); w1 = [gate | up]."""
    rng = np.random.default_rng([seed, 4])
    bound = 1.0 / np.sqrt(hidden)
    w1, w2 = [], []
    for _ in range(num_experts):
        g = rng.uniform(-bound, bound, size=(hidden, ffn))
        u = rng.uniform(-bound, bound, size=(hidden, ffn))
        w1.append(np.concatenate([g, u], axis=1))
        w2.append(rng.uniform(-bound, bound, size=(ffn, hidden)))
    return w1, w2


def init_shared_expert(hidden: int, ffn: int, seed: int) -> "ExpertWeights":
    """Builder-defined dense SwiGLU shared expert (BASELINE C4), U(+-1/sqrt(H))
    from rng([seed, 5]); replicated on every rank."""
    rng = np.random.default_rng([seed, 5])
    bound = 1.0 / np.sqrt(hidden)
    g = rng.uniform(-bound, bound, size=(hidden, ffn))
    u = rng.uniform(-bound, bound, size=(hidden, ffn))
    w2 = rng.uniform(-bound, bound, size=(ffn, hidden))
    return ExpertWeights((0,), [np.concatenate([g, u], axis=1)], [w2], ACT_SWIGLU, 0, 1)


def init_gating_matrix(hidden: int, num_experts: int, seed: int) -> np.ndarray:
    """experts.py:78-81."""
    bound = 1.0 / np.sqrt(hidden)
    return np.random.default_rng([seed, 0]).uniform(-bound, bound, size=(hidden, num_experts))


def init_expert_weights(num_experts: int, hidden: int, ffn: int, etp_size: int, seed: int,
                        ep_size: int = 1, activation: str = ACT_RELU
                        ) -> Dict[Tuple[int, int], ExpertWeights]:
    """Shard seeded expert matrices over the (ep, etp) grid -- experts.py:84-127."""
    if ffn % etp_size:
        raise ValidationError(f"ffn={ffn} is not divisible by etp_size={etp_size}",
                              constraint="etp|ffn")
    if num_experts % ep_size:
        raise ValidationError(f"num_experts={num_experts} is not divisible by ep_size={ep_size}",
                              constraint="ep|num_experts")
    if activation not in ACTIVATIONS:
        raise ValidationError(f"unknown activation {activation!r}", constraint="activation")
    if activation == ACT_SWIGLU:
        w1f, w2f = full_swiglu_matrices(num_experts, hidden, ffn, seed)
    else:
        w1f, w2f = full_expert_matrices(num_experts, hidden, ffn, seed)
    local = num_experts // ep_size
    shard = ffn // etp_size
    out = {}
    for ep_rank in range(ep_size):
        ids = tuple(range(ep_rank * local, (ep_rank + 1) * local))
        for etp_rank in range(etp_size):
            cols = slice(etp_rank * shard, (etp_rank + 1) * shard)
            if activation == ACT_SWIGLU:
                w1 = [np.concatenate([w1f[e][:, :ffn][:, cols], w1f[e][:, ffn:][:, cols]], axis=1)
                      for e in ids]
            else:
                w1 = [w1f[e][:, cols].copy() for e in ids]
            out[(ep_rank, etp_rank)] = ExpertWeights(
                expert_ids=ids, w1=w1, w2=[w2f[e][cols, :].copy() for e in ids],
                activation=activation, etp_rank=etp_rank, etp_size=etp_size)
    return out


# --------------------------------------------------------------- grouped FFN
_SIMT_WARNED = set()


def _gemm(A, B, C, **kw):
    """Grouped GEMM dispatch: tcgen05 for bf16 when available, SIMT otherwise
    (fp32 parity mode, or bf16 shapes the tensor-core kernel rejects -- the
    latter is a ~20x slower path, so it warns once per shape)."""
    from . import gemm_tc

    if A.dtype == torch.bfloat16:
        if gemm_tc.available() and gemm_tc.supports(**kw):
            return gemm_tc.gemm(A, B, C, **kw)
        key = (kw.get("N"), kw.get("K"), kw.get("M"), kw.get("grouped_dim"))
        if key not in _SIMT_WARNED:
            _SIMT_WARNED.add(key)
            warnings.warn(f"b200moe: bf16 GEMM N={key[0]} K={key[1]} M={key[2]} falls outside the tcgen05 "
                          "kernel's supported shapes (gemm_tc.supports; INTEGRATION.md §1); running the "
                          "CUDA-core SIMT GEMM", RuntimeWarning, stacklevel=3)
    return K.gemm_simt(A, B, C, **kw)


def ffn_forward(xp: torch.Tensor, goff: torch.Tensor, G: int, gexp: Optional[torch.Tensor],
                pk: PackedExperts, max_rows: int, gend: Optional[torch.Tensor] = None,
                y_scatter=None):
    """pre = xp W1_g ; h = act(pre) ; y = h W2_g  for every group g
    (experts.py:130-143 batched over groups).  Returns (pre, h, y).
    ``gend`` (optional) gives explicit group ends so groups may skip rows;
    then goff[G] must bound the last end.  ``y_scatter`` = (row_origin,
    peer_base, byte offset): y rows are stored straight into the ranks they
    came from by the GEMM epilogue (bf16 tensor-core path; y is then None)."""
    from . import gemm_tc

    R = xp.shape[0]
    H, F, N1 = pk.hidden, pk.ffn, pk.n1
    act = L.ACT_CODES[pk.act]
    dt = xp.dtype
    h = torch.empty((R, F), dtype=dt, device=xp.device)
    pre = torch.empty((R, N1), dtype=dt, device=xp.device)
    if dt == torch.bfloat16 and gemm_tc.available() and gemm_tc.fused_act_ok(pk):
        gemm_tc.ffn1_fused(xp, pk, pre, h, goff, G, gexp, max_rows, gend)
    else:
        _gemm(xp, pk.w1p, pre, grouped_dim=0, G=G, M=0, N=N1, K=H, a_sm=H, a_sk=1,
              b_sg=N1 * H, b_sk=1, b_sn=H, c_sg=0, ldc=N1, group_off=goff, group_expert=gexp,
              max_rows=max_rows, group_end=gend)
        K.act_fwd(pre, act, goff, G, F, out=h)
    if y_scatter is not None:
        gemm_tc.gemm(h, pk.w2p, None, grouped_dim=0, G=G, M=0, N=H, K=F, a_sm=F, a_sk=1, b_sg=H * F,
                     b_sk=1, b_sn=F, c_sg=0, ldc=H, group_off=goff, group_expert=gexp,
                     max_rows=max_rows, group_end=gend, scatter=y_scatter)
        return pre, h, None
    y = torch.empty((R, H), dtype=dt, device=xp.device)
    _gemm(h, pk.w2p, y, grouped_dim=0, G=G, M=0, N=H, K=F, a_sm=F, a_sk=1, b_sg=H * F, b_sk=1,
          b_sn=F, c_sg=0, ldc=H, group_off=goff, group_expert=gexp, max_rows=max_rows,
          group_end=gend)
    return pre, h, y


def ffn_forward_split(xp: torch.Tensor, goff: torch.Tensor, G: int, pk: PackedExperts, max_rows: int,
                      split, land, y_scatter):
    """ffn_forward with the first GEMM in two launches over the groups of
    ``split`` (kernels.ep_split_groups): the rows already in place (this
    rank's own), then -- after ``land()`` makes the stream wait for the rest
    of the exchange -- the received ones.  Rows are independent in GEMM1, so
    pre / h are bit-identical to one launch; GEMM2 (scatter epilogue) runs
    over the whole groups.  bf16 tensor-core path only."""
    from . import gemm_tc

    R = xp.shape[0]
    loc_off, loc_end, rem_off, rem_end, rem_exp = split
    h = torch.empty((R, pk.ffn), dtype=xp.dtype, device=xp.device)
    pre = torch.empty((R, pk.n1), dtype=xp.dtype, device=xp.device)
    gemm_tc.ffn1_fused(xp, pk, pre, h, loc_off, G, None, max_rows, loc_end)
    land()
    gemm_tc.ffn1_fused(xp, pk, pre, h, rem_off, 2 * G, rem_exp, max_rows, rem_end)
    H, F = pk.hidden, pk.ffn
    gemm_tc.gemm(h, pk.w2p, None, grouped_dim=0, G=G, M=0, N=H, K=F, a_sm=F, a_sk=1, b_sg=H * F,
                 b_sk=1, b_sn=F, c_sg=0, ldc=H, group_off=goff, max_rows=max_rows, scatter=y_scatter)
    return pre, h


def split_ok(pk: PackedExperts, dtype) -> bool:
    """Whether the split first GEMMs (ffn_forward_split / ffn_backward's
    ``split``) apply: the fused bf16 tensor-core epilogues."""
    from . import gemm_tc

    return dtype == torch.bfloat16 and gemm_tc.available() and gemm_tc.fused_act_ok(pk)


def ffn_backward(dyp: torch.Tensor, xp: torch.Tensor, pre: torch.Tensor, h: torch.Tensor,
                 goff: torch.Tensor, G: int, gexp: Optional[torch.Tensor], pk: PackedExperts,
                 max_rows: int, want_dx: bool = True, gend: Optional[torch.Tensor] = None,
                 dx_scatter=None, split=None, land=None):
    """experts.py:146-172 batched over groups: returns (dxp, dw1p, dw2p) with
    dw*p [G, ...] fp32 per GROUP (callers sum groups sharing an expert);
    dw1p[g] is [N1, H] with SwiGLU rows in [gate | up] order, so dw1p[g].T is
    the reference layout.
    ``dx_scatter``: as ffn_forward's y_scatter, for the input gradient.
    ``split`` / ``land``: as ffn_forward_split, for the first backward GEMM
    (the fused activation-derivative dgrad; requires split_ok)."""
    from . import gemm_tc

    R = dyp.shape[0]
    H, F, N1 = pk.hidden, pk.ffn, pk.n1
    act = L.ACT_CODES[pk.act]
    dt = dyp.dtype
    dev = dyp.device
    dpre = torch.empty((R, N1), dtype=dt, device=dev)
    if split is not None:
        loc_off, loc_end, rem_off, rem_end, rem_exp = split
        gemm_tc.dgrad2_fused(dyp, pk, pre, dpre, loc_off, G, None, max_rows, loc_end)
        land()
        gemm_tc.dgrad2_fused(dyp, pk, pre, dpre, rem_off, 2 * G, rem_exp, max_rows, rem_end)
    elif dt == torch.bfloat16 and gemm_tc.available() and gemm_tc.fused_act_ok(pk):
        gemm_tc.dgrad2_fused(dyp, pk, pre, dpre, goff, G, gexp, max_rows, gend)
    else:
        dh = torch.empty((R, F), dtype=dt, device=dev)
        _gemm(dyp, pk.w2p, dh, grouped_dim=0, G=G, M=0, N=F, K=H, a_sm=H, a_sk=1, b_sg=H * F,
              b_sk=F, b_sn=1, c_sg=0, ldc=F, group_off=goff, group_expert=gexp, max_rows=max_rows,
              group_end=gend)
        K.act_bwd(dh, pre, act, goff, G, F, out=dpre)
    dxp = None
    if dx_scatter is not None:
        gemm_tc.gemm(dpre, pk.w1p, None, grouped_dim=0, G=G, M=0, N=H, K=N1, a_sm=N1, a_sk=1,
                     b_sg=N1 * H, b_sk=H, b_sn=1, c_sg=0, ldc=H, group_off=goff, group_expert=gexp,
                     max_rows=max_rows, group_end=gend, scatter=dx_scatter)
    elif want_dx:
        dxp = torch.empty((R, H), dtype=dt, device=dev)
        _gemm(dpre, pk.w1p, dxp, grouped_dim=0, G=G, M=0, N=H, K=N1, a_sm=N1, a_sk=1,
              b_sg=N1 * H, b_sk=H, b_sn=1, c_sg=0, ldc=H, group_off=goff, group_expert=gexp,
              max_rows=max_rows, group_end=gend)
    dw2p = torch.empty((G, H, F), dtype=torch.float32, device=dev)
    _gemm(dyp, h, dw2p, grouped_dim=1, G=G, M=H, N=F, K=0, a_sm=1, a_sk=H, b_sg=0, b_sk=F,
          b_sn=1, c_sg=H * F, ldc=F, group_off=goff, max_rows=max_rows, group_end=gend)
    dw1p = torch.empty((G, N1, H), dtype=torch.float32, device=dev)
    kw = dict(grouped_dim=1, G=G, M=N1, N=H, K=0, a_sm=1, a_sk=N1, b_sg=0, b_sk=H, b_sn=1,
              c_sg=N1 * H, ldc=H, group_off=goff, max_rows=max_rows, group_end=gend)
    glu = pk.act == "swiglu"
    if glu and dt == torch.bfloat16 and gemm_tc.available() and gemm_tc.supports(**kw):
        # the epilogue stores the packed SwiGLU rows de-interleaved ([gate | up])
        gemm_tc.gemm(dpre, xp, dw1p, glu_f=F, **kw)
    else:
        _gemm(dpre, xp, dw1p, **kw)
        if glu:
            b = dw1p.view(G, F // 32, 2, 32, H)
            dw1p = torch.cat([b[:, :, 0].reshape(G, F, H), b[:, :, 1].reshape(G, F, H)], dim=1)
    return dxp, dw1p, dw2p


def _single_group(n: int, device) -> torch.Tensor:
    return torch.tensor([0, n], dtype=torch.int32, device=device)


def expert_forward_shard(tokens, weights: ExpertWeights, expert_id: int, dtype=None):
    """Partial FFN output of one expert shard -- experts.py:130-143.

    ``tokens`` is a CUDA tensor (fp32 or bf16; numpy is moved to CUDA fp32).
    Returns (out, cache) with cache = (tokens, pre) like the reference (``pre``
    is in the packed column order for SwiGLU)."""
    i = weights.local_index(expert_id)
    x = tokens if isinstance(tokens, torch.Tensor) else torch.as_tensor(np.asarray(tokens, np.float64), dtype=torch.float32)
    if not x.is_cuda:
        x = x.cuda()
    dt = dtype or x.dtype
    x = x.to(dt).contiguous()
    pk = weights.packed(dt, x.device)
    sub = PackedExperts(pk.w1p[i:i + 1], pk.w2p[i:i + 1], pk.act, pk.hidden, pk.ffn)
    goff = _single_group(x.shape[0], x.device)
    pre, h, y = ffn_forward(x, goff, 1, None, sub, x.shape[0])
    return y, (x, pre)


def expert_backward_shard(upstream, cache, weights: ExpertWeights, expert_id: int):
    """Gradients through one expert shard -- experts.py:146-172.

    Returns (partial token grad, w1 shard grad, w2 shard grad) with weight
    grads in the reference layout ([H, N1] and [F, H], fp32)."""
    i = weights.local_index(expert_id)
    x, pre = cache
    u = upstream if isinstance(upstream, torch.Tensor) else torch.as_tensor(np.asarray(upstream, np.float64))
    u = u.to(device=x.device, dtype=x.dtype).contiguous()
    pk = weights.packed(x.dtype, x.device)
    if tuple(u.shape) != (x.shape[0], pk.hidden):
        raise ValidationError(
            f"upstream shape {tuple(u.shape)} does not match forward output ({x.shape[0]}, {pk.hidden})",
            constraint="upstream-shape")
    sub = PackedExperts(pk.w1p[i:i + 1], pk.w2p[i:i + 1], pk.act, pk.hidden, pk.ffn)
    goff = _single_group(x.shape[0], x.device)
    h = K.act_fwd(pre, L.ACT_CODES[pk.act], goff, 1, pk.ffn)
    dxp, dw1p, dw2p = ffn_backward(u, x, pre, h, goff, 1, None, sub, x.shape[0])
    return dxp, unpack_w1_grad(dw1p, pk.act)[0], unpack_w2_grad(dw2p)[0]
