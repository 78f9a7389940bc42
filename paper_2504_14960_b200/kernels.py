"""Torch-tensor wrappers over the C ABI (one function per entry point).

Every wrapper launches on the current CUDA stream, allocates outputs with the
torch caching allocator, and never synchronises.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import torch

from . import _lib as L
from .errors import ValidationError

# rows per expert segment in the padded (GEMM) layout: a multiple of the
# GEMM's 64-row K block (the weight-gradient GEMMs walk each expert's rows as
# K); B200MOE_GEMM_ALIGN overrides (experiments; 64 or 128)
GEMM_ALIGN = int(os.environ.get("B200MOE_GEMM_ALIGN", "128"))
if GEMM_ALIGN not in (64, 128, 256):
    raise ValidationError(f"B200MOE_GEMM_ALIGN={GEMM_ALIGN} must be 64, 128 or 256", constraint="gemm-align")


def _cuda(t: torch.Tensor, name: str, dtype=None) -> torch.Tensor:
    if not t.is_cuda:
        raise ValidationError(f"{name} must be a CUDA tensor", constraint=f"{name}-cuda")
    if dtype is not None and t.dtype != dtype:
        raise ValidationError(f"{name} must be {dtype}, got {t.dtype}", constraint=f"{name}-dtype")
    if not t.is_contiguous():
        raise ValidationError(f"{name} must be contiguous", constraint=f"{name}-contiguous")
    return t


def _sp():
    return L.stream_ptr()


_ROWS_CACHE = {}


def _single_group(rows: int, device) -> torch.Tensor:
    """Device [0, rows] int32 (one GEMM group spanning all rows), cached."""
    key = (rows, str(device))
    t = _ROWS_CACHE.get(key)
    if t is None:
        t = torch.tensor([0, rows], dtype=torch.int32).pin_memory().to(device, non_blocking=True)
        _ROWS_CACHE[key] = t
    return t


def dense_gemm(A, B, C, *, M: int, N: int, K: int, a_sm, a_sk, b_sk, b_sn, ldc, accumulate=False):
    """C (+)= A @ B on CUDA cores in fp32 (mixed input dtypes allowed): the
    skinny router GEMMs (x W_g, dz W_g^T) when E is too large for the fused
    warp kernels."""
    return gemm_simt(A, B, C, grouped_dim=0, G=1, M=M, N=N, K=K, a_sm=a_sm, a_sk=a_sk, b_sg=0,
                     b_sk=b_sk, b_sn=b_sn, c_sg=0, ldc=ldc, group_off=_single_group(M, A.device),
                     max_rows=M, accumulate=accumulate)


def _ep(E: int) -> int:
    return (E + 7) // 8 * 8


def _tc_router(x: torch.Tensor, parts) -> bool:
    """Tensor-core router GEMMs: bf16 tokens, W_g parts given, tcgen05 on."""
    from . import gemm_tc

    return parts is not None and x.dtype == torch.bfloat16 and gemm_tc.available() and x.shape[1] % 8 == 0


def split_bf16x3(src: torch.Tensor, want3: bool = True, want6: bool = False):
    """fp32 [rows, E] -> bf16 (hi | mid | lo) [rows, 3Ep] and/or
    (hi | hi | hi | mid | mid | lo) [rows, 6Ep]."""
    rows, E = src.shape
    _cuda(src, "src", torch.float32)
    o3 = torch.empty((rows, 3 * _ep(E)), dtype=torch.bfloat16, device=src.device) if want3 else None
    o6 = torch.empty((rows, 6 * _ep(E)), dtype=torch.bfloat16, device=src.device) if want6 else None
    L.call("b200moe_split_bf16x3", L.ptr(src), rows, E, L.ptr(o3), L.ptr(o6), _sp())
    return o3, o6


def sum_parts(parts: torch.Tensor, G: int, rows: int, E: int) -> torch.Tensor:
    out = torch.empty((rows, E), dtype=torch.float32, device=parts.device)
    L.call("b200moe_sum_parts", L.ptr(parts), G, rows, E, L.ptr(out), _sp())
    return out


def router_logits(x: torch.Tensor, w_g: torch.Tensor, parts=None) -> torch.Tensor:
    """logits = x @ W_g (router.py:145) in fp32.  bf16 tokens with ``parts``
    (GatingParams.device_w_g_parts): one tensor-core GEMM against the three
    exact bf16 parts of W_g, then the parts are folded in fixed order."""
    T, H = x.shape
    E = w_g.shape[1]
    _cuda(x, "x")
    _cuda(w_g, "w_g", torch.float32)
    if T > 0 and _tc_router(x, parts):
        from . import gemm_tc

        w3t = parts[0]
        n3 = w3t.shape[0]
        l3 = torch.empty((T, n3), dtype=torch.float32, device=x.device)
        gemm_tc.gemm(x, w3t, l3, grouped_dim=0, G=1, M=0, N=n3, K=H, a_sm=H, a_sk=1, b_sg=0, b_sk=1,
                     b_sn=H, c_sg=0, ldc=n3, group_off=_single_group(T, x.device), max_rows=T,
                     tag="router_tc")
        return sum_parts(l3, 1, T, E)
    out = torch.empty((T, E), dtype=torch.float32, device=x.device)
    if E > 8 and T > 0:
        # tiled fp32 GEMM (64x64 tiles) instead of the per-token warp kernel
        return dense_gemm(x, w_g, out, M=T, N=E, K=H, a_sm=H, a_sk=1, b_sk=E, b_sn=1, ldc=E)
    L.call("b200moe_router_logits", L.ptr(x), L.dtype_code(x.dtype), L.ptr(w_g), T, H, E,
           L.ptr(out), _sp())
    return out


def router_term(dz: torch.Tensor, w_g: torch.Tensor, out: torch.Tensor, parts=None) -> torch.Tensor:
    """out += dz @ w_g^T  (dispatcher.py:490).  bf16 ``out`` with ``parts``:
    one tensor-core GEMM over K = 6Ep (the six significant part products of
    dz and W_g), reduce-added into out; otherwise a tiled fp32 GEMM."""
    T, E = dz.shape
    H = w_g.shape[0]
    if T == 0:
        return out
    if _tc_router(out, parts):
        from . import gemm_tc

        _, dz6 = split_bf16x3(dz, want3=False, want6=True)
        w6 = parts[1]
        k6 = w6.shape[1]
        return gemm_tc.gemm(dz6, w6, out, grouped_dim=0, G=1, M=0, N=H, K=k6, a_sm=k6, a_sk=1, b_sg=0,
                            b_sk=1, b_sn=k6, c_sg=0, ldc=H, group_off=_single_group(T, dz.device),
                            max_rows=T, accumulate=True, tag="router_tc")
    return dense_gemm(dz, w_g, out, M=T, N=H, K=E, a_sm=E, a_sk=1, b_sk=1, b_sn=E, ldc=H,
                      accumulate=True)


_SPLITK_CACHE = {}


def _splitk_groups(T: int, device, parts: int = 8) -> Tuple[torch.Tensor, int]:
    """Token-chunk offsets (multiples of 64, last = T) for a split-K GEMM."""
    key = (T, str(device), parts)
    if key not in _SPLITK_CACHE:
        c = max(64, ((T + parts - 1) // parts + 63) // 64 * 64)
        offs = list(range(0, T, c)) + [T]
        t = torch.tensor(offs, dtype=torch.int32).pin_memory().to(device, non_blocking=True)
        _SPLITK_CACHE[key] = (t, len(offs) - 1)
    return _SPLITK_CACHE[key]


def router_stats(topk_idx: torch.Tensor, kept, scores, E: int):
    """-> (counts [E] int64, top1 [E] int64, score_sum [E] fp64) on the device."""
    T, k = topk_idx.shape
    dev = topk_idx.device
    ws = torch.empty((max(int(L.load().b200moe_router_stats_ws(T, E)), 8),), dtype=torch.uint8, device=dev)
    counts = torch.empty((E,), dtype=torch.int64, device=dev)
    top1 = torch.empty((E,), dtype=torch.int64, device=dev)
    psum = torch.empty((E,), dtype=torch.float64, device=dev)
    kept_u8 = None if kept is None else kept.to(torch.uint8).contiguous()
    L.call("b200moe_router_stats", L.ptr(topk_idx), L.ptr(kept_u8), L.ptr(scores), T, k, E,
           L.ptr(counts), L.ptr(top1), L.ptr(psum), L.ptr(ws), ctypes.c_size_t(ws.numel()), _sp())
    return counts, top1, psum


def router_topk(logits: torch.Tensor, k: int, gate_fn: int, renorm: bool, want_f64: bool = False,
                status: Optional[torch.Tensor] = None):
    T, E = logits.shape
    _cuda(logits, "logits", torch.float32)
    dev = logits.device
    scores = torch.empty((T, E), dtype=torch.float32, device=dev)
    idx = torch.empty((T, k), dtype=torch.int32, device=dev)
    gates = torch.empty((T, k), dtype=torch.float32, device=dev)
    g64 = torch.empty((T, k), dtype=torch.float64, device=dev) if want_f64 else None
    L.call("b200moe_router_topk", L.ptr(logits), T, E, k, gate_fn, int(renorm), L.ptr(scores),
           L.ptr(idx), L.ptr(gates), L.ptr(g64), L.ptr(status), _sp())
    return scores, idx, gates, g64


def router_fwd_supported(x: torch.Tensor, E: int) -> bool:
    """The fused tensor-core router forward: bf16 tokens, E <= 64, H % 8 == 0."""
    from . import gemm_tc

    return (x.dtype == torch.bfloat16 and x.shape[1] % 8 == 0 and x.shape[1] >= 64
            and int(L.load().b200moe_router_fwd_tc_np(E)) > 0 and gemm_tc.available())


def router_fwd(x: torch.Tensor, w_tc: torch.Tensor, E: int, k: int, gate_fn: int, renorm: bool,
               status: torch.Tensor, want_f64: bool = False):
    """Fused router forward (router.py:141-162): logits on the tensor cores
    against the exact bf16 parts of W_g (``w_tc``, GatingParams.device_w_g_tc),
    softmax/sigmoid and top-k in the same kernel.  Non-finite logits set bit 0
    of ``status``.  -> (logits, scores, idx, gates, gates_f64)"""
    T, H = x.shape
    _cuda(x, "x", torch.bfloat16)
    _cuda(w_tc, "w_tc", torch.bfloat16)
    dev = x.device
    logits = torch.empty((T, E), dtype=torch.float32, device=dev)
    scores = torch.empty((T, E), dtype=torch.float32, device=dev)
    idx = torch.empty((T, k), dtype=torch.int32, device=dev)
    gates = torch.empty((T, k), dtype=torch.float32, device=dev)
    g64 = torch.empty((T, k), dtype=torch.float64, device=dev) if want_f64 else None
    L.call("b200moe_router_fwd_tc", L.ptr(x), T, H, L.ptr(w_tc), E, k, gate_fn, int(renorm),
           L.ptr(logits), L.ptr(scores), L.ptr(idx), L.ptr(gates), L.ptr(g64), L.ptr(status), _sp())
    return logits, scores, idx, gates, g64


class PlanTensors:
    """Device outputs of one b200moe_dispatch_plan call."""

    __slots__ = ("kept", "counts", "offsets", "poffsets", "send_row", "gemm_row", "perm",
                 "perm_gates", "T", "k", "E", "align")

    def __init__(self, **kw):
        for k_, v in kw.items():
            setattr(self, k_, v)


def dispatch_plan(topk_idx: torch.Tensor, gates: torch.Tensor, E: int, cap: int = 0,
                  kept_in: Optional[torch.Tensor] = None, order: Optional[torch.Tensor] = None,
                  align: int = GEMM_ALIGN, want_perm_gates: bool = True) -> PlanTensors:
    T, k = topk_idx.shape
    dev = topk_idx.device
    _cuda(topk_idx, "topk_idx", torch.int32)
    lib = L.load()
    ws_bytes = int(lib.b200moe_dispatch_plan_ws(T, E))
    ws = torch.empty((max(ws_bytes, 4),), dtype=torch.uint8, device=dev)
    kept = torch.empty((T, k), dtype=torch.uint8, device=dev)
    counts = torch.empty((E,), dtype=torch.int32, device=dev)
    offsets = torch.empty((E + 1,), dtype=torch.int32, device=dev)
    poffsets = torch.empty((E + 1,), dtype=torch.int32, device=dev)
    send_row = torch.empty((T, k), dtype=torch.int32, device=dev)
    gemm_row = torch.empty((T, k), dtype=torch.int32, device=dev)
    perm = torch.empty((max(T * k, 1),), dtype=torch.int64, device=dev)
    pg = torch.empty((max(T * k, 1),), dtype=torch.float32, device=dev) if want_perm_gates else None
    L.call("b200moe_dispatch_plan", L.ptr(topk_idx), L.ptr(gates), L.ptr(kept_in), L.ptr(order),
           T, k, E, int(cap), align, L.ptr(ws), ctypes.c_size_t(ws.numel()), L.ptr(kept),
           L.ptr(counts), L.ptr(offsets), L.ptr(poffsets), L.ptr(send_row), L.ptr(gemm_row),
           L.ptr(perm), L.ptr(pg), _sp())
    return PlanTensors(kept=kept, counts=counts, offsets=offsets, poffsets=poffsets,
                       send_row=send_row, gemm_row=gemm_row, perm=perm, perm_gates=pg, T=T, k=k,
                       E=E, align=align)


def capacity_by_gate(plan0: PlanTensors, gates64: torch.Tensor, positions: Optional[torch.Tensor],
                     cap: int) -> torch.Tensor:
    T, k, E = plan0.T, plan0.k, plan0.E
    kept = torch.zeros((T, k), dtype=torch.uint8, device=gates64.device)
    L.call("b200moe_capacity_by_gate", L.ptr(plan0.perm), L.ptr(plan0.offsets), L.ptr(gates64),
           L.ptr(positions), T, k, E, int(cap), L.ptr(kept), _sp())
    return kept


def permute(x: torch.Tensor, pair_row: torch.Tensor, out_rows: int, scale=None,
            poffsets=None, counts=None, E: int = 0, align: int = GEMM_ALIGN,
            out: Optional[torch.Tensor] = None) -> torch.Tensor:
    T, H = x.shape
    k = pair_row.shape[1]
    _cuda(x, "x")
    if out is None:
        out = torch.empty((max(out_rows, 1), H), dtype=x.dtype, device=x.device)
    L.call("b200moe_permute", L.ptr(x), L.dtype_code(x.dtype), T, H, k, L.ptr(pair_row),
           L.ptr(scale), L.ptr(out), L.ptr(poffsets), L.ptr(counts), E, align, _sp())
    return out


def permute_bwd(u: torch.Tensor, pair_row: torch.Tensor, gates: torch.Tensor,
                y_rows: torch.Tensor, poffsets=None, counts=None, E: int = 0,
                align: int = GEMM_ALIGN) -> Tuple[torch.Tensor, torch.Tensor]:
    T, H = u.shape
    k = pair_row.shape[1]
    _cuda(u, "upstream")
    if u.dtype != y_rows.dtype:
        raise ValidationError("upstream and expert rows must share a dtype", constraint="dtype")
    dy = torch.empty_like(y_rows)
    dg = torch.empty((T, k), dtype=torch.float32, device=u.device)
    L.call("b200moe_permute_bwd", L.ptr(u), L.dtype_code(u.dtype), T, H, k, L.ptr(pair_row),
           L.ptr(gates), L.ptr(y_rows), L.ptr(dy), L.ptr(dg), L.ptr(poffsets), L.ptr(counts), E,
           align, _sp())
    return dy, dg


def combine(rows: torch.Tensor, pair_row: torch.Tensor, T: int, gates=None, dz=None, w_gT=None,
            out: Optional[torch.Tensor] = None, out_dtype=None, accumulate: bool = False,
            rows_out: Optional[torch.Tensor] = None):
    """``rows`` [R, H], or [P, R, H] ETP partial rows (summed in fp32 in
    member order inside the combine, b200moe_combine_parts; ``rows_out``
    then receives the reduced pair rows)."""
    if rows.dim() == 3:
        P_, R, H = rows.shape
        k = pair_row.shape[1]
        fused = (rows.dtype == torch.bfloat16 and H % 8 == 0 and k <= 8 and (dz is None or dz.shape[1] <= 8)
                 and (out is None or out.dtype == torch.bfloat16) and out_dtype in (None, torch.bfloat16))
        if not fused:
            red = ep_reduce_parts(rows)
            if rows_out is not None:
                rows_out.copy_(red)
            return combine(red, pair_row, T, gates=gates, dz=dz, w_gT=w_gT, out=out, out_dtype=out_dtype,
                           accumulate=accumulate)
        if out is None:
            out = torch.empty((T, H), dtype=rows.dtype, device=rows.device)
        E = 0 if dz is None else dz.shape[1]
        L.call("b200moe_combine_parts", L.ptr(rows), P_, R * H, L.ptr(rows_out), T, H, k, L.ptr(pair_row),
               L.ptr(gates), L.ptr(dz), L.ptr(w_gT), E, L.ptr(out), int(accumulate), _sp())
        return out
    H = rows.shape[1]
    k = pair_row.shape[1]
    if out is None:
        out = torch.empty((T, H), dtype=out_dtype or rows.dtype, device=rows.device)
    E = 0 if dz is None else dz.shape[1]
    L.call("b200moe_combine", L.ptr(rows), L.dtype_code(rows.dtype), T, H, k, L.ptr(pair_row),
           L.ptr(gates), L.ptr(dz), L.ptr(w_gT), E, L.ptr(out), L.dtype_code(out.dtype),
           int(accumulate), _sp())
    return out


def router_bwd(dgates, scores, topk_idx, gates, gate_fn: int, renorm: bool, want_parts: bool = False):
    """dz [T, E] fp32 (dispatcher.py:470-488); with ``want_parts`` also
    (dz, parts): the exact bf16 split of dz laid out for router_wgrad_tc."""
    T, E = scores.shape
    k = topk_idx.shape[1]
    dz = torch.empty((T, E), dtype=torch.float32, device=scores.device)
    parts = None
    if want_parts:
        nb = int(L.load().b200moe_router_parts_cols(E))
        parts = torch.empty((T, nb), dtype=torch.bfloat16, device=scores.device)
    L.call("b200moe_router_bwd", L.ptr(dgates), L.ptr(scores), L.ptr(topk_idx), L.ptr(gates), T,
           E, k, gate_fn, int(renorm), L.ptr(dz), L.ptr(parts), _sp())
    return (dz, parts) if want_parts else dz


def router_wgrad_tc_supported(x: torch.Tensor, E: int) -> bool:
    from . import gemm_tc

    return (x.dtype == torch.bfloat16 and x.shape[1] % 64 == 0 and x.shape[1] >= 128
            and int(L.load().b200moe_router_parts_cols(E)) > 0 and gemm_tc.available())


def router_wgrad_tc(x: torch.Tensor, dz_parts: torch.Tensor, E: int) -> torch.Tensor:
    """dW_g = x^T dz (dispatcher.py:489) on the tensor cores against the dz
    parts of router_bwd(want_parts=True); x read once."""
    T, H = x.shape
    _cuda(x, "x", torch.bfloat16)
    _cuda(dz_parts, "dz_parts", torch.bfloat16)
    dwg = torch.empty((H, E), dtype=torch.float32, device=x.device)
    ws_bytes = int(L.load().b200moe_router_wgrad_tc_ws(T, H, E))
    ws = torch.empty((max(ws_bytes // 4, 1),), dtype=torch.float32, device=x.device)
    L.call("b200moe_router_wgrad_tc", L.ptr(x), L.ptr(dz_parts), T, H, E, L.ptr(dwg), L.ptr(ws),
           ctypes.c_size_t(ws.numel() * 4), _sp())
    return dwg


def router_wgrad(x: torch.Tensor, dz: torch.Tensor, tc: bool = False) -> torch.Tensor:
    """dW_g = x^T dz (dispatcher.py:489).  ``tc`` (bf16 x): one split-K
    tensor-core GEMM against dz's three exact bf16 parts, folded in fixed
    order; otherwise the deterministic split-K CUDA-core kernels."""
    T, H = x.shape
    E = dz.shape[1]
    if tc and T > 0 and _tc_router(x, ()):
        from . import gemm_tc

        dz3, _ = split_bf16x3(dz)
        n3 = dz3.shape[1]
        goff, G = _splitk_groups(T, x.device)
        part = torch.empty((G, H, n3), dtype=torch.float32, device=x.device)
        gemm_tc.gemm(x, dz3, part, grouped_dim=1, G=G, M=H, N=n3, K=0, a_sm=1, a_sk=H, b_sg=0,
                     b_sk=n3, b_sn=1, c_sg=H * n3, ldc=n3, group_off=goff, max_rows=T,
                     tag="router_tc")
        return sum_parts(part, G, H, E)
    dwg = torch.empty((H, E), dtype=torch.float32, device=x.device)
    ws_bytes = int(L.load().b200moe_router_wgrad_ws(T, H, E))
    ws = torch.empty((max(ws_bytes // 4, 1),), dtype=torch.float32, device=x.device)
    L.call("b200moe_router_wgrad", L.ptr(x), L.dtype_code(x.dtype), L.ptr(dz), T, H, E,
           L.ptr(dwg), L.ptr(ws), ctypes.c_size_t(ws.numel() * 4), _sp())
    return dwg


def gemm_simt(A, B, C, *, grouped_dim: int, G: int, M: int, N: int, K: int, a_sm, a_sk, b_sg,
              b_sk, b_sn, c_sg, ldc, group_off, group_expert=None, max_rows: int = 0,
              accumulate: bool = False, group_end=None):
    args = L.GemmArgs(
        dtype_in=L.dtype_code(A.dtype), dtype_out=L.dtype_code(C.dtype), grouped_dim=grouped_dim,
        accumulate=int(accumulate), G=G, M=M, N=N, K=K,
        A=L.ptr(A), a_sm=a_sm, a_sk=a_sk, B=L.ptr(B), b_sg=b_sg, b_sk=b_sk, b_sn=b_sn,
        C=L.ptr(C), c_sg=c_sg, ldc=ldc, group_off=L.ptr(group_off),
        group_expert=L.ptr(group_expert), max_rows=max_rows, dtype_b=L.dtype_code(B.dtype),
        group_end=L.ptr(group_end))
    L.call("b200moe_gemm_simt", ctypes.byref(args), _sp())
    return C


def act_fwd(pre, act: int, group_off, G: int, F: int, out=None):
    rows = pre.shape[0]
    if out is None:
        out = torch.empty((rows, F), dtype=pre.dtype, device=pre.device)
    L.call("b200moe_act_fwd", L.ptr(pre), L.dtype_code(pre.dtype), act, L.ptr(group_off), G, rows,
           F, L.ptr(out), _sp())
    return out


# ------------------------------------------------ EP exchange over peer memory
# peer_base: int64 device tensor [ep] with the base address of every EP
# member's symmetric buffer (peer.PeerExchange owns it and the region offsets).
def ep_counts_push(counts: torch.Tensor, me: int, ep: int, peer_base, cnt_off: int, status=None):
    _cuda(counts, "counts", torch.int32)
    L.call("b200moe_ep_counts_push", L.ptr(counts), me, ep, counts.numel(), L.ptr(peer_base),
           cnt_off, L.ptr(status), _sp())


def ep_barrier(peer_base, flag_off: int, me: int, ep: int, epoch: int):
    L.call("b200moe_ep_barrier", L.ptr(peer_base), flag_off, me, ep, epoch & 0xFFFFFFFF, _sp())


def ep_layout(cnt: torch.Tensor, me: int, ep: int, etp: int, L_: int, align: int, cap_rows: int,
              status=None):
    """-> (seg_off [ep*L], goff [L+1], gcount [L]) int32 on the device."""
    dev = cnt.device
    seg_off = torch.empty((ep * L_,), dtype=torch.int32, device=dev)
    goff = torch.empty((L_ + 1,), dtype=torch.int32, device=dev)
    gcount = torch.empty((L_,), dtype=torch.int32, device=dev)
    L.call("b200moe_ep_layout", L.ptr(cnt), me, ep, etp, L_, align, cap_rows, L.ptr(seg_off),
           L.ptr(goff), L.ptr(gcount), L.ptr(status), _sp())
    return seg_off, goff, gcount


def ep_zero_pads(buf: torch.Tensor, goff, gcount, G: int, align: int, origin=None):
    _cuda(buf, "receive buffer", torch.bfloat16)
    L.call("b200moe_ep_zero_pads", L.ptr(buf), buf.shape[1], L.ptr(goff), L.ptr(gcount), G, align,
           L.ptr(origin), _sp())


def ep_dispatch(x: torch.Tensor, topk_idx, gemm_row, poffsets, seg_off, L_: int, peer_base, me: int,
                etp: int, dst_off: int, origin_off: int = 0, bwd: bool = False, y_rows=None,
                gates=None, dup_off: int = -1, status=None, part: int = 0, dgates=None):
    """Forward: push x rows to the owners' receive buffers and record their
    origin.  Backward: push gates*u rows; returns dgates [T, k] fp32 = <u, y>
    with y the returned expert outputs (``y_rows``, local padded layout).
    ``dup_off >= 0``: one push per (token, EP index), duplicates recorded in
    the receivers' dup tables (resolved by ``ep_expand``).
    ``part`` 1 / 2: only the stores into this rank's own / the other members'
    buffers (b200moe_ep_dispatch_part); the two parts of a backward share one
    ``dgates`` tensor (each writes its own pairs)."""
    T, H = x.shape
    k = topk_idx.shape[1]
    _cuda(x, "x", torch.bfloat16)
    dg = dgates
    if bwd and dg is None:
        dg = torch.empty((T, k), dtype=torch.float32, device=x.device)
    if part == 0:
        L.call("b200moe_ep_dispatch", L.ptr(x), T, H, k, L_, L.ptr(topk_idx), L.ptr(gemm_row),
               L.ptr(poffsets), L.ptr(seg_off), L.ptr(peer_base), me, etp, dst_off, origin_off, dup_off,
               L.ptr(y_rows), L.ptr(gates), L.ptr(dg), int(bwd), L.ptr(status), _sp())
    else:
        L.call("b200moe_ep_dispatch_part", L.ptr(x), T, H, k, L_, L.ptr(topk_idx), L.ptr(gemm_row),
               L.ptr(poffsets), L.ptr(seg_off), L.ptr(peer_base), me, etp, dst_off, origin_off, dup_off,
               L.ptr(y_rows), L.ptr(gates), L.ptr(dg), int(bwd), int(part), L.ptr(status), _sp(),
               tag="ep_dispatch" if part == 2 else "ep_dispatch_local")
    return dg


def ep_split_groups(cnt: torch.Tensor, me: int, ep: int, etp: int, L_: int, seg_off, goff, gcount):
    """-> (loc_off [L+1], loc_end [L], rem_off [2L+1], rem_end [2L], rem_exp [2L]) int32 views: the
    groups of the first GEMM split into the rows this rank sent itself and the rest."""
    split = torch.empty((8 * L_ + 2,), dtype=torch.int32, device=cnt.device)
    L.call("b200moe_ep_split_groups", L.ptr(cnt), me, ep, etp, L_, L.ptr(seg_off), L.ptr(goff),
           L.ptr(gcount), L.ptr(split), _sp())
    n = L_
    return (split[:n + 1], split[n + 1:2 * n + 1], split[2 * n + 1:4 * n + 2], split[4 * n + 2:6 * n + 2],
            split[6 * n + 2:8 * n + 2])


def ep_expand(buf: torch.Tensor, goff, gcount, G: int, dup: torch.Tensor, phase: int):
    """Resolve the deduplicated rows of a receive buffer (phase 0 forward;
    1 then 2 backward)."""
    _cuda(buf, "receive buffer", torch.bfloat16)
    L.call("b200moe_ep_expand", L.ptr(buf), buf.shape[1], L.ptr(goff), L.ptr(gcount), G, L.ptr(dup),
           phase, _sp())


def ep_reduce_parts(parts: torch.Tensor) -> torch.Tensor:
    """[P, rows, H] bf16 partial rows -> [rows, H] bf16, summed in fp32."""
    P_, rows, H = parts.shape
    out = torch.empty((rows, H), dtype=parts.dtype, device=parts.device)
    L.call("b200moe_ep_reduce_parts", L.ptr(parts), P_, rows * H, rows * H, L.ptr(out), _sp())
    return out


def act_bwd(dh, pre, act: int, group_off, G: int, F: int, out=None):
    rows = pre.shape[0]
    if out is None:
        out = torch.empty_like(pre)
    L.call("b200moe_act_bwd", L.ptr(dh), L.ptr(pre), L.dtype_code(pre.dtype), act,
           L.ptr(group_off), G, rows, F, L.ptr(out), _sp())
    return out


def fullseq_capacity(seg_sorted: torch.Tensor, order: torch.Tensor, cap: int, k: int,
                     pos_by_pos: Optional[torch.Tensor] = None, status: Optional[torch.Tensor] = None):
    """Kept flags (uint8, original slot order) of a full-sequence capacity pass
    over device-sorted pair keys (router.py:209-269); see b200moe.h."""
    N = seg_sorted.numel()
    _cuda(seg_sorted, "seg_sorted", torch.int64)
    _cuda(order, "order", torch.int64)
    kept = torch.empty((N,), dtype=torch.uint8, device=seg_sorted.device)
    L.call("b200moe_fullseq_capacity", L.ptr(seg_sorted), L.ptr(order), N, int(cap), L.ptr(kept),
           L.ptr(pos_by_pos), k, L.ptr(status), _sp())
    return kept
