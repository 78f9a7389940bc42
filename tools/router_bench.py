"""Time the router kernels (forward logits/top-k and backward dz, dz.W_g^T,
x^T dz) at the C2 / C4 per-GPU shapes, in isolation, CUDA events on the
launching stream, L2 flushed before every rep.  Prints one JSON line per
variant: mean us and the algorithmic GB/s of the x read.

  python tools/router_bench.py [--config c2|c4] [--reps 20]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2504_14960_b200 import _lib as L  # noqa: E402
from paper_2504_14960_b200 import kernels as K  # noqa: E402
from paper_2504_14960_b200.router import GatingParams  # noqa: E402

SHAPES = {"c2": (16384, 4096, 8, 2), "c4": (16384, 3584, 64, 8)}


def timeit(fn, reps, flush, batch=4):
    """Mean/min us per call of ``batch`` back-to-back calls (the GPU never
    waits for the host between them; the operands exceed or nearly fill the
    126 MB L2, which is flushed before every batch)."""
    ts = []
    for i in range(reps + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()  # queue ahead so e0 is not followed by a host-side gap
        e0.record()
        for _ in range(batch):
            fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3 / batch)
    return (sum(ts) / len(ts), min(ts)) if ts else (0.0, 0.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=sorted(SHAPES))
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    T, H, E, k = SHAPES[a.config]
    dev = torch.device("cuda", 0)
    L.load()
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
    wg = (torch.rand((H, E), generator=g, device=dev) * 2 - 1) / H ** 0.5
    params = GatingParams(w_g=wg, k=k)
    parts = params.device_w_g_parts(dev)
    wgT = params.device_w_gT(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    xbytes = T * H * 2
    res = []

    def rec(name, fn, nbytes=xbytes):
        mean, best = timeit(fn, a.reps, flush)
        res.append(dict(config=a.config, op=name, us=round(mean, 2), us_min=round(best, 2),
                        gbs=round(nbytes / (mean * 1e-6) / 1e9, 1)))
        print(json.dumps(res[-1]), flush=True)

    rec("logits_tc+sum_parts", lambda: K.router_logits(x, wg, parts=parts))
    rec("logits_cuda_core", lambda: K.router_logits(x, wg))
    logits = K.router_logits(x, wg)
    rec("topk", lambda: K.router_topk(logits, k, L.GATE_SOFTMAX, False), T * E * 8)
    st = torch.zeros((1,), dtype=torch.int32, device=dev)
    w_tc = params.device_w_g_tc(dev)
    rec("router_fwd_fused", lambda: K.router_fwd(x, w_tc, E, k, L.GATE_SOFTMAX, False, st))
    scores, idx, gates, _ = K.router_topk(logits, k, L.GATE_SOFTMAX, False)
    dgates = torch.randn((T, k), generator=g, device=dev)
    rec("router_bwd", lambda: K.router_bwd(dgates, scores, idx, gates, L.GATE_SOFTMAX, False), T * E * 8)
    dz = K.router_bwd(dgates, scores, idx, gates, L.GATE_SOFTMAX, False)
    rec("router_bwd+parts", lambda: K.router_bwd(dgates, scores, idx, gates, L.GATE_SOFTMAX, False,
                                                  want_parts=True), T * E * 8)
    _, dzp = K.router_bwd(dgates, scores, idx, gates, L.GATE_SOFTMAX, False, want_parts=True)
    rec("wgrad_tc_fused", lambda: K.router_wgrad_tc(x, dzp, E))
    rec("wgrad_tc", lambda: K.router_wgrad(x, dz, tc=True))
    rec("wgrad_cuda_core", lambda: K.router_wgrad(x, dz, tc=False))
    out = torch.zeros((T, H), dtype=torch.bfloat16, device=dev)
    rec("router_term_tc", lambda: K.router_term(dz, wg, out, parts=parts), 2 * xbytes)
    # combine backward (k pair rows -> token row) with and without dz . W_g^T
    R = T * k
    rows = torch.randn((R, H), generator=g, device=dev).to(torch.bfloat16)
    pair_row = torch.randperm(R, generator=g, device=dev).to(torch.int32).reshape(T, k).contiguous()
    cb = (R + T) * H * 2
    rec("combine_bwd", lambda: K.combine(rows, pair_row, T), cb)
    if E <= 8:
        rec("combine_bwd+dz.W_gT", lambda: K.combine(rows, pair_row, T, dz=dz, w_gT=wgT), cb)


if __name__ == "__main__":
    main()
