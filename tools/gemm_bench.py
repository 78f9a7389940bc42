"""Time the six expert GEMMs of one C2 step in isolation (CUDA events).

    python tools/gemm_bench.py [--rows 32768] [--experts 8] [--reps 5]

Env toggles of the kernel (read per launch): B200MOE_CTA_GROUP=1|2,
B200MOE_DEBUG_NOSTORE=1 (skip epilogue stores: mainloop only).
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_14960_b200 as B  # noqa: E402
from paper_2504_14960_b200 import gemm_tc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=32768)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--burst", type=int, default=20, help="back-to-back launches per timing")
    ap.add_argument("--variants", default="",
                    help="comma list of ENV=VAL[;ENV=VAL] settings timed interleaved, e.g. "
                         "'B200MOE_STORE_HINT=0,B200MOE_STORE_HINT=1'")
    ap.add_argument("--routed", action="store_true", help="uneven groups from a real routing")
    ap.add_argument("--splitk", type=int, default=4, help="K slices of the split-K dgrad1 variant")
    ap.add_argument("--only", default="", help="run only the GEMMs whose name contains this")
    ap.add_argument("--wait-prof", action="store_true",
                    help="library built with -DB200MOE_WAIT_PROF: print per-role barrier wait shares")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    R, E, H, F = a.rows, a.experts, a.hidden, a.ffn
    g = torch.Generator(device=dev).manual_seed(0)
    bnd = H ** -0.5
    w1 = [(torch.rand((H, 2 * F), generator=g, device=dev) * 2 - 1) * bnd for _ in range(E)]
    w2 = [(torch.rand((F, H), generator=g, device=dev) * 2 - 1) * bnd for _ in range(E)]
    pk = B.ExpertWeights(tuple(range(E)), w1, w2, "swiglu", 0, 1).packed(torch.bfloat16, dev)
    del w1, w2
    if a.routed:
        # group sizes of a real top-2 routing of R/2 tokens (128-row padded layout)
        from paper_2504_14960_b200 import kernels as K

        T = R // 2
        xt = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
        wg = ((torch.rand((H, E), generator=g, device=dev) * 2 - 1) * bnd).float()
        _, idx, gates, _ = K.router_topk(K.router_logits(xt, wg), 2, 0, False)
        plan = K.dispatch_plan(idx, gates, E)
        goff = plan.poffsets
        R = int(goff[-1])
        print("routed groups:", [int(v) for v in plan.counts], "rows", R)
    else:
        goff = torch.arange(0, R + 1, R // E, dtype=torch.int32, device=dev)
    x = torch.randn((R, H), generator=g, device=dev).to(torch.bfloat16)
    dy = torch.randn((R, H), generator=g, device=dev).to(torch.bfloat16)
    pre = torch.empty((R, 2 * F), dtype=torch.bfloat16, device=dev)
    h = torch.empty((R, F), dtype=torch.bfloat16, device=dev)
    y = torch.empty((R, H), dtype=torch.bfloat16, device=dev)
    dpre = torch.empty_like(pre)
    dx = torch.empty_like(x)
    dw2 = torch.empty((E, H, F), dtype=torch.float32, device=dev)
    dw1 = torch.empty((E, 2 * F, H), dtype=torch.float32, device=dev)
    N1 = 2 * F
    fl_small = 2.0 * R * H * F
    dx32 = torch.empty((R, H), dtype=torch.float32, device=dev)

    def dgrad1_split(S):
        # experiment: split K = N1 into S slices so one slice's operand
        # panels of an expert fit L2; fp32 partials reduce-added by TMA
        ks = N1 // S
        for s in range(S):
            gemm_tc.gemm(dpre[:, s * ks:(s + 1) * ks], pk.w1p[:, s * ks:(s + 1) * ks, :], dx32,
                         grouped_dim=0, G=E, M=0, N=H, K=ks, a_sm=N1, a_sk=1, b_sg=N1 * H, b_sk=H,
                         b_sn=1, c_sg=0, ldc=H, group_off=goff, max_rows=R, accumulate=s > 0)

    _w1t = {}

    def w1t():
        if "t" not in _w1t:
            _w1t["t"] = pk.w1p.transpose(1, 2).contiguous()
        return _w1t["t"]

    runs = [
        ("fwd1 swiglu", 2 * fl_small, lambda: gemm_tc.ffn1_fused(x, pk, pre, h, goff, E, None, R)),
        ("fwd2 store", fl_small, lambda: gemm_tc.gemm(
            h, pk.w2p, y, grouped_dim=0, G=E, M=0, N=H, K=F, a_sm=F, a_sk=1, b_sg=H * F, b_sk=1,
            b_sn=F, c_sg=0, ldc=H, group_off=goff, max_rows=R)),
        ("dgrad2 swiglu_bwd", fl_small, lambda: gemm_tc.dgrad2_fused(dy, pk, pre, dpre, goff, E, None, R)),
        ("dgrad1 store", 2 * fl_small, lambda: gemm_tc.gemm(
            dpre, pk.w1p, dx, grouped_dim=0, G=E, M=0, N=H, K=N1, a_sm=N1, a_sk=1, b_sg=N1 * H,
            b_sk=H, b_sn=1, c_sg=0, ldc=H, group_off=goff, max_rows=R)),
        ("dgrad1 splitK", 2 * fl_small, lambda: dgrad1_split(a.splitk)),
        # experiment: W1 as a K-major B operand (a transposed copy [E, H, N1])
        ("dgrad1 kmajorB", 2 * fl_small, lambda: gemm_tc.gemm(
            dpre, w1t(), dx, grouped_dim=0, G=E, M=0, N=H, K=N1, a_sm=N1, a_sk=1, b_sg=N1 * H,
            b_sk=1, b_sn=N1, c_sg=0, ldc=H, group_off=goff, max_rows=R)),
        ("wgrad2 f32", fl_small, lambda: gemm_tc.gemm(
            dy, h, dw2, grouped_dim=1, G=E, M=H, N=F, K=0, a_sm=1, a_sk=H, b_sg=0, b_sk=F, b_sn=1,
            c_sg=H * F, ldc=F, group_off=goff, max_rows=R)),
        ("wgrad1 f32", 2 * fl_small, lambda: gemm_tc.gemm(
            dpre, x, dw1, grouped_dim=1, G=E, M=N1, N=H, K=0, a_sm=1, a_sk=N1, b_sg=0, b_sk=H,
            b_sn=1, c_sg=N1 * H, ldc=H, group_off=goff, max_rows=R)),
    ]
    if a.only:
        runs = [r for r in runs if a.only in r[0]]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    variants = [v for v in a.variants.split(",") if v] or [""]

    def apply(v):
        for kv in filter(None, v.split(";")):
            k_, val = kv.split("=")
            os.environ[k_] = val

    import threading

    import pynvml

    pynvml.nvmlInit()
    hdl = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    samples = []
    stop = threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(hdl) / 1000.0))
            time.sleep(0.005)

    if a.wait_prof:
        import ctypes

        from paper_2504_14960_b200 import _lib

        lib = _lib.load()
        buf = (ctypes.c_ulonglong * 8)()
        for name, fl, fn in runs:
            fn()
            lib.b200moe_debug_wait_prof(buf, 1)
            fn()
            lib.b200moe_debug_wait_prof(buf, 1)
            w = list(buf)
            mma_life = max(w[2], 1)
            epi_life = max(w[5], 1)
            print(f"{name:20s} MMA waits: operands {w[0] / mma_life:6.1%}  accumulator {w[1] / mma_life:6.1%} | "
                  f"producer waits for a stage {w[3] / 2 / mma_life:6.1%} | epilogue waits: accumulator "
                  f"{w[4] / epi_life:6.1%}  pre chunk {w[6] / epi_life:6.1%} | MMA CTAs {w[7]}", flush=True)
        return

    tot = {v: [0.0, 0.0] for v in variants}
    for name, fl, fn in runs:
        for v in variants:
            apply(v)
            fn()
        torch.cuda.synchronize()
        res = {v: [] for v in variants}
        for _ in range(a.reps):
            for v in variants:  # interleaved so clock drift hits every variant alike
                apply(v)
                samples.clear()
                stop.clear()
                th = threading.Thread(target=sampler)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.burst):  # back-to-back, long enough for NVML to see the clock
                    fn()
                e1.record()
                th.start()
                torch.cuda.synchronize()
                stop.set()
                th.join()
                clk = sorted(c for c, _ in samples)
                pw = sorted(p_ for _, p_ in samples)
                res[v].append((e0.elapsed_time(e1) / a.burst, clk[len(clk) // 2] if clk else 0,
                               pw[len(pw) // 2] if pw else 0))
        for v in variants:
            r = sorted(res[v])[len(res[v]) // 2]
            tot[v][0] += r[0]
            tot[v][1] += fl
            print(f"{name:20s} {v:32s} {r[0]:8.3f} ms  {fl / r[0] / 1e9:7.1f} TF/s  "
                  f"sm {r[1]} MHz  {r[2]:.0f} W", flush=True)
    for v in variants:
        print(f"{'total':20s} {v:32s} {tot[v][0]:8.3f} ms  {tot[v][1] / tot[v][0] / 1e9:7.1f} TF/s",
              flush=True)

if __name__ == "__main__":
    main()
