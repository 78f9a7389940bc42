"""ctypes binding of libb200moe.so (the C ABI declared in include/b200moe.h).

There is no CPU fallback: importing the package works without a GPU (so the
host-side logic can be tested on CPU), but every compute entry point raises
if the shared library is missing or no sm_100 device is present.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

from .errors import ValidationError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libb200moe.so")

OK, EINVAL, ELAUNCH, EUNSUPPORTED, ENODEV = 0, 1, 2, 3, 4
F32, BF16 = 0, 1
GATE_SOFTMAX, GATE_SIGMOID = 0, 1
ACT_RELU, ACT_GELU, ACT_SWIGLU = 0, 1, 2
ACT_CODES = {"relu": ACT_RELU, "gelu": ACT_GELU, "swiglu": ACT_SWIGLU}
MAJOR_K, MAJOR_MN = 0, 1

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int
SZ = ctypes.c_size_t


class GemmArgs(ctypes.Structure):
    """Mirror of b200moe_gemm_args."""

    _fields_ = [
        ("dtype_in", I32), ("dtype_out", I32), ("grouped_dim", I32), ("accumulate", I32),
        ("G", I32), ("M", I64), ("N", I64), ("K", I64),
        ("A", P), ("a_sm", I64), ("a_sk", I64),
        ("B", P), ("b_sg", I64), ("b_sk", I64), ("b_sn", I64),
        ("C", P), ("c_sg", I64), ("ldc", I64),
        ("group_off", P), ("group_expert", P), ("max_rows", I64), ("dtype_b", I32),
        ("group_end", P),
    ]


# name -> argtypes (restype is int unless listed in _RESTYPES)
_SIGS = {
    "b200moe_version": [],
    "b200moe_last_error": [],
    "b200moe_device_check": [],
    "b200moe_enable_peer_access": [I32],
    "b200moe_router_logits": [P, I32, P, I64, I64, I32, P, P],
    "b200moe_router_topk": [P, I64, I32, I32, I32, I32, P, P, P, P, P, P],
    "b200moe_router_fwd_tc_np": [I32],
    "b200moe_router_fwd_tc": [P, I64, I64, P, I32, I32, I32, I32, P, P, P, P, P, P, P],
    "b200moe_dispatch_plan_ws": [I64, I32],
    "b200moe_dispatch_plan": [P, P, P, P, I64, I32, I32, I64, I32, P, SZ, P, P, P, P, P, P, P, P, P],
    "b200moe_capacity_by_gate": [P, P, P, P, I64, I32, I32, I64, P, P],
    "b200moe_router_bwd": [P, P, P, P, I64, I32, I32, I32, I32, P, P, P],
    "b200moe_router_parts_cols": [I32],
    "b200moe_fullseq_capacity": [P, P, I64, I64, P, P, I32, P, P],
    "b200moe_router_wgrad_tc_ws": [I64, I64, I32],
    "b200moe_router_wgrad_tc": [P, P, I64, I64, I32, P, P, SZ, P],
    "b200moe_router_wgrad_ws": [I64, I64, I32],
    "b200moe_router_wgrad": [P, I32, P, I64, I64, I32, P, P, SZ, P],
    "b200moe_permute": [P, I32, I64, I64, I32, P, P, P, P, P, I32, I32, P],
    "b200moe_permute_bwd": [P, I32, I64, I64, I32, P, P, P, P, P, P, P, I32, I32, P],
    "b200moe_combine": [P, I32, I64, I64, I32, P, P, P, P, I32, P, I32, I32, P],
    "b200moe_gemm_simt": [ctypes.POINTER(GemmArgs), P],
    "b200moe_gemm_tc": [P, P],  # argtypes refined in gemm_tc.py
    "b200moe_act_fwd": [P, I32, I32, P, I32, I64, I64, P, P],
    "b200moe_act_bwd": [P, P, I32, I32, P, I32, I64, I64, P, P],
    "b200moe_split_bf16x3": [P, I64, I32, P, P, P],
    "b200moe_router_stats_ws": [I64, I32],
    "b200moe_router_stats": [P, P, P, I64, I32, I32, P, P, P, P, SZ, P],
    "b200moe_sum_parts": [P, I64, I64, I32, P, P],
    "b200moe_ep_counts_push": [P, I32, I32, I32, P, I64, P, P],
    "b200moe_ep_barrier": [P, I64, I32, I32, ctypes.c_uint32, P],
    "b200moe_ep_layout": [P, I32, I32, I32, I32, I32, I64, P, P, P, P, P],
    "b200moe_ep_reduce_parts": [P, I32, I64, I64, P, P],
    "b200moe_ep_zero_pads": [P, I64, P, P, I32, I32, P, P],
    "b200moe_ep_dispatch": [P, I64, I64, I32, I32, P, P, P, P, P, I32, I32, I64, I64, I64, P, P, P, I32, P, P],
    "b200moe_ep_dispatch_part": [P, I64, I64, I32, I32, P, P, P, P, P, I32, I32, I64, I64, I64, P, P, P, I32,
                                 I32, P, P],
    "b200moe_ep_split_groups": [P, I32, I32, I32, I32, P, P, P, P, P],
    "b200moe_combine_parts": [P, I32, I64, P, I64, I64, I32, P, P, P, P, I32, P, I32, P],
    "b200moe_ep_expand": [P, I64, P, P, I32, P, I32, P],
}
_RESTYPES = {
    "b200moe_version": ctypes.c_char_p,
    "b200moe_last_error": ctypes.c_char_p,
    "b200moe_dispatch_plan_ws": SZ,
    "b200moe_router_wgrad_ws": SZ,
    "b200moe_router_stats_ws": SZ,
    "b200moe_router_wgrad_tc_ws": SZ,
}

_lib: Optional[ctypes.CDLL] = None
_device_ok = False


def exported_symbols():
    """Names every binding expects the library to export (checked on CPU)."""
    return sorted(_SIGS)


def load(check_device: bool = True) -> ctypes.CDLL:
    """Load the library (once).  Raises RuntimeError loudly when missing."""
    global _lib, _device_ok
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not found: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
    if check_device and not _device_ok:
        rc = _lib.b200moe_device_check()
        if rc != OK:
            raise RuntimeError("b200moe: " + _lib.b200moe_last_error().decode())
        _device_ok = True
    return _lib


def check(rc: int, what: str) -> None:
    if rc == OK:
        return
    msg = f"{what}: " + load(False).b200moe_last_error().decode()
    if rc == EINVAL:
        raise ValidationError(msg, constraint=what)
    raise RuntimeError(msg)


# kernels launched per entry point (bench.py reports the total as gpu_launches)
_LAUNCHES = {"b200moe_dispatch_plan": 3}
_LAUNCHES["b200moe_router_wgrad"] = 2
_LAUNCHES["b200moe_router_wgrad_tc"] = 2
_LAUNCHES["b200moe_router_stats"] = 2
_NO_LAUNCH = {"b200moe_version", "b200moe_last_error", "b200moe_device_check", "b200moe_enable_peer_access",
              "b200moe_router_fwd_tc_np", "b200moe_router_parts_cols", "b200moe_router_wgrad_tc_ws",
              "b200moe_dispatch_plan_ws", "b200moe_router_wgrad_ws", "b200moe_router_stats_ws"}
_launches = 0


def note_launches(n: int) -> None:
    global _launches
    _launches += n


def reset_launch_count() -> None:
    global _launches
    _launches = 0


def launch_count() -> int:
    return _launches


class Profile:
    """Optional CUDA-event timing around every launching C-ABI call (bench)."""

    def __init__(self):
        self.on = False
        self.events = []

    def enable(self):
        self.on, self.events = True, []

    def disable(self):
        self.on = False

    def begin(self):
        import torch

        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def end(self, name, e0):
        import torch

        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        self.events.append((name, e0, e1))

    def collect(self):
        """[(name, ms)] plus the span from the first start to the last end."""
        import torch

        torch.cuda.synchronize()
        per = [(n, a.elapsed_time(b)) for n, a, b in self.events]
        span = self.events[0][1].elapsed_time(self.events[-1][2]) if self.events else 0.0
        return per, span


PROFILE = Profile()


def call(name: str, *args, tag: Optional[str] = None) -> None:
    lib = load()
    e0 = PROFILE.begin() if PROFILE.on and name not in _NO_LAUNCH else None
    check(getattr(lib, name)(*args), name)
    if e0 is not None:
        PROFILE.end(tag or name.replace("b200moe_", ""), e0)
    if name not in _NO_LAUNCH:
        n = _LAUNCHES.get(name, 1)
        if name in ("b200moe_permute", "b200moe_permute_bwd") and args[-5]:
            n += 1  # alignment-padding zero kernel
        if name == "b200moe_router_fwd_tc" and args[4] > 32:
            n += 1  # the warp-per-token top-k follows the tensor-core logits
        note_launches(n)


def ptr(t) -> Optional[int]:
    """Device pointer of a tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def dtype_code(dtype) -> int:
    import torch

    if dtype == torch.float32:
        return F32
    if dtype == torch.bfloat16:
        return BF16
    raise ValidationError(f"unsupported dtype {dtype}", constraint="dtype")
