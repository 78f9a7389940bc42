"""tcgen05 / TMEM / TMA grouped GEMM (bf16 in, fp32 accumulate) -- wrapper of
b200moe_gemm_tc (csrc/gemm_tc.cu).

The expert FFN calls it with fused epilogues: GEMM1 writes the bf16
pre-activations and the activation in one pass (SwiGLU or relu/gelu), the
backward dgrad of GEMM2 applies the activation derivative in its epilogue.
Set B200MOE_DISABLE_TC=1 to force the SIMT kernel (cross-checks only).
"""
from __future__ import annotations

import ctypes
import os

from . import _lib as L

EPI_STORE, EPI_SWIGLU_FWD, EPI_SWIGLU_BWD, EPI_ACT_FWD, EPI_ACT_BWD, EPI_SCATTER = range(6)
MAX_GROUPS = 512  # csrc/gemm_tc.cu MAX_G
P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int


class TcGemmArgs(ctypes.Structure):
    """Mirror of b200moe_tc_gemm_args."""

    _fields_ = [
        ("G", I32), ("grouped_dim", I32), ("M", I64), ("N", I64), ("K", I64),
        ("A", P), ("a_major", I32), ("lda", I64), ("a_rows", I64),
        ("B", P), ("b_major", I32), ("ldb", I64), ("b_batch", I64), ("b_batch_stride", I64),
        ("C", P), ("ldc", I64), ("c_sg", I64), ("out_dtype", I32), ("accumulate", I32),
        ("group_off", P), ("group_expert", P),
        ("epilogue", I32), ("act", I32), ("H", P), ("ldh", I64), ("PRE", P), ("ldpre", I64),
        ("num_ctas", I32), ("group_end", P),
        ("row_origin", P), ("peer_base", P), ("scatter_off", I64), ("glu_f", I64),
    ]


_registered = False


def _lib():
    global _registered
    lib = L.load()
    if not _registered:
        lib.b200moe_gemm_tc.argtypes = [ctypes.POINTER(TcGemmArgs), P]
        lib.b200moe_gemm_tc.restype = ctypes.c_int
        _registered = True
    return lib


def available() -> bool:
    return os.environ.get("B200MOE_DISABLE_TC", "0") != "1"


def _ok8(*vals) -> bool:
    return all(int(v) % 8 == 0 for v in vals)


def supports(**kw) -> bool:
    """Whether a SIMT-style argument set maps onto the tensor-core kernel."""
    if not 1 <= int(kw.get("G", 1)) <= MAX_GROUPS:
        return False
    if kw["grouped_dim"] == 0:
        if kw["a_sk"] != 1:
            return False
        if kw["b_sk"] == 1:
            ok_b = _ok8(kw["b_sn"])
        elif kw["b_sn"] == 1:
            ok_b = _ok8(kw["b_sk"])
        else:
            return False
        return ok_b and _ok8(kw["a_sm"], kw["N"], kw["K"])
    return (kw["a_sm"] == 1 and kw["b_sn"] == 1 and _ok8(kw["a_sk"], kw["b_sk"], kw["M"], kw["N"]))


_EPI_NAMES = {EPI_STORE: "store", EPI_SWIGLU_FWD: "swiglu_fwd", EPI_SWIGLU_BWD: "swiglu_bwd",
              EPI_ACT_FWD: "act_fwd", EPI_ACT_BWD: "act_bwd", EPI_SCATTER: "scatter"}


def _run(args: TcGemmArgs, tag: str = "gemm_tc") -> None:
    lib = _lib()
    prof = L.PROFILE
    e0 = prof.begin() if prof.on else None
    L.check(lib.b200moe_gemm_tc(ctypes.byref(args), L.stream_ptr()), "b200moe_gemm_tc")
    L.note_launches(1)
    if e0 is not None:
        kind = "wgrad" if args.grouped_dim == 1 else _EPI_NAMES[args.epilogue]
        prof.end(f"{tag}[{kind} N={args.N} K={args.K} M={args.M}]", e0)


def gemm(A, B, C, *, grouped_dim, G, M, N, K, a_sm, a_sk, b_sg, b_sk, b_sn, c_sg, ldc, group_off,
         group_expert=None, max_rows=0, accumulate=False, group_end=None, scatter=None,
         tag="gemm_tc", glu_f=0):
    """Same argument convention as kernels.gemm_simt.  ``scatter`` =
    (row_origin, peer_base, byte_offset): bf16 rows go to the ranks they came
    from instead of C (C may be None; ldc is the destination row length)."""
    a = TcGemmArgs()
    a.G, a.grouped_dim, a.M, a.N, a.K = G, grouped_dim, M, N, K
    a.A, a.a_rows = L.ptr(A), A.shape[0]
    if grouped_dim == 0:
        a.a_major, a.lda = L.MAJOR_K, a_sm
        a.b_batch = B.shape[0] if B.dim() == 3 else 1
        a.b_batch_stride = b_sg
        if b_sk == 1:
            a.b_major, a.ldb = L.MAJOR_K, b_sn
        else:
            a.b_major, a.ldb = L.MAJOR_MN, b_sk
    else:
        a.a_major, a.lda = L.MAJOR_MN, a_sk
        a.b_major, a.ldb, a.b_batch, a.b_batch_stride = L.MAJOR_MN, b_sk, 1, 0
    a.B = L.ptr(B)
    a.C, a.ldc, a.c_sg = L.ptr(C), ldc, c_sg
    a.out_dtype = L.dtype_code(C.dtype) if C is not None else L.BF16
    a.accumulate = int(accumulate)
    a.group_off, a.group_expert = L.ptr(group_off), L.ptr(group_expert)
    a.group_end = L.ptr(group_end)
    a.epilogue = EPI_STORE
    a.glu_f = glu_f
    if scatter is not None:
        a.epilogue = EPI_SCATTER
        a.row_origin, a.peer_base, a.scatter_off = L.ptr(scatter[0]), L.ptr(scatter[1]), scatter[2]
    _run(a, tag)
    return C


def fused_act_ok(pk) -> bool:
    H, F, N1 = pk.hidden, pk.ffn, pk.n1
    if not _ok8(H, F, N1):
        return False
    if pk.act == "swiglu":
        return N1 % 64 == 0 and F % 32 == 0
    return True


def ffn1_fused(xp, pk, pre, h, goff, G, gexp, max_rows, gend=None):
    """pre = xp W1_g (bf16) and h = act(pre) in one tensor-core pass."""
    a = TcGemmArgs()
    H, F, N1 = pk.hidden, pk.ffn, pk.n1
    a.G, a.grouped_dim, a.M, a.N, a.K = G, 0, 0, N1, H
    a.A, a.a_major, a.lda, a.a_rows = L.ptr(xp), L.MAJOR_K, H, xp.shape[0]
    a.B, a.b_major, a.ldb = L.ptr(pk.w1p), L.MAJOR_K, H
    a.b_batch, a.b_batch_stride = pk.w1p.shape[0], N1 * H
    a.C, a.ldc, a.c_sg, a.out_dtype = L.ptr(pre), N1, 0, L.BF16
    a.group_off, a.group_expert = L.ptr(goff), L.ptr(gexp)
    a.group_end = L.ptr(gend)
    if pk.act == "swiglu":
        a.epilogue = EPI_SWIGLU_FWD
    else:
        a.epilogue, a.act = EPI_ACT_FWD, L.ACT_CODES[pk.act]
    a.H, a.ldh = L.ptr(h), F
    _run(a)


def dgrad2_fused(dyp, pk, pre, dpre, goff, G, gexp, max_rows, gend=None):
    """dpre = (dy W2_g^T) * act'(pre) in one tensor-core pass."""
    a = TcGemmArgs()
    H, F, N1 = pk.hidden, pk.ffn, pk.n1
    a.G, a.grouped_dim, a.M, a.N, a.K = G, 0, 0, F, H
    a.A, a.a_major, a.lda, a.a_rows = L.ptr(dyp), L.MAJOR_K, H, dyp.shape[0]
    # W2p [L, H, F] is B = (k=h, n=f) stored K x N with N contiguous: MN-major
    a.B, a.b_major, a.ldb = L.ptr(pk.w2p), L.MAJOR_MN, F
    a.b_batch, a.b_batch_stride = pk.w2p.shape[0], H * F
    a.C, a.ldc, a.c_sg, a.out_dtype = L.ptr(dpre), N1, 0, L.BF16
    a.group_off, a.group_expert = L.ptr(goff), L.ptr(gexp)
    a.group_end = L.ptr(gend)
    if pk.act == "swiglu":
        a.epilogue = EPI_SWIGLU_BWD
    else:
        a.epilogue, a.act = EPI_ACT_BWD, L.ACT_CODES[pk.act]
    a.PRE, a.ldpre = L.ptr(pre), N1
    _run(a)
