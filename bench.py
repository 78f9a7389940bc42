"""MoE-layer fwd+bwd benchmark (BASELINE.json metric) on B200.

Workload (N=1): Mixtral-8x7B MoE layer shape -- 8 experts top-2, hidden 4096,
expert FFN 14336 (SwiGLU), 16384 tokens per GPU, dropless, bf16 -- all 8
experts on the one GPU (EP=1).  N>1 (torchrun, one rank per GPU): EP=N with
16384 tokens per GPU (weak scaling); the EP exchange is device-side over NVLink
peer memory: a push kernel sends token rows to the expert owners and the second
GEMM's epilogue stores the outputs back (B200MOE_EP_EXCHANGE=nccl: NCCL
all-to-all-v).

A step = router -> dispatch -> grouped SwiGLU FFN -> combine, then the full
backward (input, router and expert weight gradients).  Synthetic N(0,1)
tokens and U(+-1/sqrt(H)) weights (the reference's init distributions).

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle port
(numpy float64, the reference's algorithm) on a bounded token sample instead.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer fwd+bwd tokens/s"
# experiments only: B200MOE_E2E_CHECK=0 times the e2e leg without input validation
E2E_CHECK = os.environ.get("B200MOE_E2E_CHECK", "1") != "0"
UNIT = "tokens/s"

# BASELINE.json configs[1..4] (configs[0] is the CPU-oracle case); per-GPU
# token counts from SURVEY.md §8.  etp applies when n_gpus >= 2.
CONFIGS = {
    "c2": dict(name="Mixtral-8x7B MoE layer (C2)", E=8, k=2, H=4096, F=14336, T=16384, cf=None,
               shared=0, etp=1, pad=False),
    "c3": dict(name="Mixtral-8x7B, CF=1.0 pad-to-capacity, EP x ETP2 (C3)", E=8, k=2, H=4096,
               F=14336, T=16384, cf=1.0, shared=0, etp=2, pad=True),
    "c4": dict(name="Qwen2-57B-A14B MoE layer + shared expert (C4)", E=64, k=8, H=3584, F=2560,
               T=16384, cf=None, shared=20480, etp=1, pad=False),
    "c5": dict(name="Mixtral-8x22B MoE layer, seq 32K over TP2xCP2 (C5)", E=8, k=2, H=6144,
               F=16384, T=8192, cf=None, shared=0, etp=1, pad=False),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS),
                    help="BASELINE.json config (default c2, the metric's headline)")
    ap.add_argument("--tokens", type=int, default=None, help="tokens per GPU (override)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile-only", action="store_true",
                    help="a few steps, no extra legs (for ncu)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock, power and throttle reasons polled through NVML every 10 ms
    from a thread while the timed region runs (nvidia-smi as a fallback)."""

    # NVML clocks-event reason bits
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (t, sm_mhz, max_mhz, power_w, reason_bits)
        self.window = None  # (t0, t1) wall-clock of the timed region
        self.stop_ev = threading.Event()
        self.err = None

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def _handle(self, nv):
        import torch

        try:
            prop = torch.cuda.get_device_properties(self.index)
            bus = f"{prop.pci_domain_id:08x}:{prop.pci_bus_id:02x}:{prop.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:  # noqa: BLE001
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = self._handle(nv)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self.stop_ev.is_set():
                self.rows.append((time.time(), nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx,
                                  nv.nvmlDeviceGetPowerUsage(h) / 1000.0, int(get_reasons(h))))
                time.sleep(0.01)
        except Exception as exc:  # noqa: BLE001
            self.err = f"nvml unavailable: {exc}"

    def start(self):
        self.thread = threading.Thread(target=self._poll, daemon=True)
        self.thread.start()

    def stop(self):
        self.stop_ev.set()
        self.thread.join(timeout=5)
        rows = self.rows
        if self.window is not None:
            rows = [r for r in rows if self.window[0] <= r[0] <= self.window[1]] or rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no samples"]}
        sm = sorted(r[1] for r in rows)
        pw = sorted(r[3] for r in rows)
        bits = 0
        for r in rows:
            bits |= r[4]
        reasons = sorted(name for bit, name in self.REASONS.items() if bits & bit)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": rows[0][2], "reasons": reasons,
                "samples": len(rows), "sm_mhz_min": sm[0], "power_w_median": pw[len(pw) // 2]}


def traffic(config: str):
    """DRAM bytes per step of the expert GEMMs from the committed ncu --set
    full capture (profiles/traffic.json), or None for configs not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f).get(config)
        return None if d is None else {"dram_bytes_per_step": d["gemm_tc_dram_bytes_per_step"],
                                       "algorithmic_bytes_per_step": d["gemm_tc_algorithmic_bytes_per_step"],
                                       "source": d["source"]}
    except (OSError, KeyError, ValueError):
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d.get("bf16_tflops", 1665.1), d.get("bf16_tflops_sustained", 1401.1), d.get("hbm_gbs", 6536.0), "measured"
    except OSError:
        return 1590.0, 1400.0, 6650.0, "fallback"


# ------------------------------------------------------------- CPU baseline
def cpu_reference_sample(a, n_tokens: int, reps: int = 1, warm: int = 0):
    """Time the CPU oracle (numpy float64 restatement of the reference's
    moe_forward + moe_backward) on `n_tokens` tokens at full H/F/k width.
    Only k experts are materialised (every token routes to both), which keeps
    the per-token work of the full config while bounding host memory."""
    import numpy as np

    from oracle import moe_oracle as O

    threads = os.cpu_count() or 1
    H, F, k = a.hidden, a.ffn, a.topk
    E = k
    rng = np.random.default_rng(0)
    b = 1.0 / np.sqrt(H)
    experts = []
    for _ in range(E):
        w1 = rng.uniform(-b, b, size=(H, 2 * F))
        w2 = rng.uniform(-b, b, size=(F, H))
        experts.append(O.Expert(w1, w2, "swiglu"))
    wg = rng.uniform(-b, b, size=(H, E))
    cfg = O.LayerConfig(k=k)
    x = rng.standard_normal((n_tokens, H))
    u = rng.standard_normal((n_tokens, H))
    times = []
    for i in range(warm + reps):
        t0 = time.perf_counter()
        y, st = O.layer_forward(x, x @ wg, experts, cfg)
        O.layer_backward(u, st, experts, cfg, w_g=wg)
        dt = time.perf_counter() - t0
        if i >= warm:
            times.append(dt)
    return n_tokens / (sum(times) / len(times)), threads, times


REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def moefold_sample(a, n_ranks: int, n_tokens: int, reps: int, warm: int):
    """Time the UNMODIFIED reference (oracle/_ref/moefold, installed from
    /root/reference by oracle/Makefile): moe_forward + moe_backward
    (dispatcher.py:246-510) over SimWorld(n_ranks) on ``n_tokens`` tokens in
    total, at the config's full E/k/H/F and its EP x ETP mesh.  The reference's
    experts are ReLU MLPs (it has no SwiGLU and no shared expert), with its
    own init distributions (experts.py:66-81; weights built per shard directly
    to bound host memory and init time, which is excluded).  Returns
    (tokens/s, threads, per-step seconds, ms of weight init) or None when the
    reference is not installed."""
    if not os.path.isdir(os.path.join(REF_DIR, "moefold")):
        return None
    import numpy as np

    threads = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import moefold as M

    c = a.cfg
    etp = c["etp"] if n_ranks >= 2 else 1
    ep = max(1, n_ranks // etp)
    E, k, H, F = c["E"], c["k"], c["H"], c["F"]
    topo = M.ParallelTopology(world_size=n_ranks, ep=ep, etp=etp, tp=etp)
    t0 = time.perf_counter()
    params = M.GatingParams(w_g=M.init_gating_matrix(H, E, 0), k=k, capacity_factor=c["cf"])
    rng = np.random.default_rng([0, 1])
    b = 1.0 / np.sqrt(H)
    L_, Fs = E // ep, F // etp
    weights = {}
    for e_i in range(ep):
        ids = tuple(range(e_i * L_, (e_i + 1) * L_))
        for t_i in range(etp):
            weights[(e_i, t_i)] = M.ExpertWeights(
                ids, [rng.uniform(-b, b, size=(H, Fs)) for _ in ids],
                [rng.uniform(-b, b, size=(Fs, H)) for _ in ids], "relu", t_i, etp)
    per = max(1, n_tokens // n_ranks)
    xr = np.random.default_rng([0, 2])
    blocks = [M.TokenBlock(xr.standard_normal((per, H)), np.arange(r * per, (r + 1) * per))
              for r in range(n_ranks)]
    ups = [np.random.default_rng([0, 3, r]).standard_normal((per, H)) for r in range(n_ranks)]
    init_ms = (time.perf_counter() - t0) * 1e3
    times = []
    for i in range(warm + reps):
        t0 = time.perf_counter()
        world = M.SimWorld(n_ranks)
        _, fctx = M.moe_forward(blocks, weights, topo, params, world, seq_len=per)
        M.moe_backward(ups, fctx)
        dt = time.perf_counter() - t0
        if i >= warm:
            times.append(dt)
    return per * n_ranks / (sum(times) / len(times)), threads, times, init_ms


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_ranks = int(os.environ.get("WORLD_SIZE", a.gpus))
    # a bounded slice per step (~2-4 s of 16-core work at Mixtral width), so
    # the default 20+5-step run ends within a few minutes
    n_tok = 512 if a.hidden * a.ffn >= 4096 * 14336 else 1024
    got = moefold_sample(a, n_ranks, n_tok, reps=a.steps, warm=a.warmup)
    if got is not None:
        tok_s, threads, times, init_ms = got
        sample = (f"{n_tok} tokens/step over SimWorld({n_ranks}) at E{a.experts} top-{a.topk} "
                  f"H={a.hidden} F={a.ffn} (ReLU: the reference has no SwiGLU"
                  + (", no shared expert" if a.cfg["shared"] else "") +
                  f"), moefold.moe_forward+moe_backward from oracle/_ref (unmodified reference, "
                  f"numpy float64, OpenBLAS {threads} threads, {cpu_model()}); weight init "
                  f"{init_ms:.0f} ms excluded")
        kind = "reference"
    else:
        n_tok = 128
        tok_s, threads, times = cpu_reference_sample(a, n_tok, reps=a.steps, warm=a.warmup)
        sample = (f"{n_tok} tokens/step at H={a.hidden} F={a.ffn} SwiGLU top-{a.topk} (k experts "
                  f"materialised), numpy float64 oracle port, {threads} threads "
                  f"(oracle/_ref missing)")
        kind = "port"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": tok_s, "unit": UNIT,
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1000.0 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(a),
        "cpu_baseline": {"value": tok_s, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample, "source": "oracle/_ref/moefold" if kind == "reference"
                         else "oracle/moe_oracle.py"},
        "e2e": {"value": tok_s, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def resolve(a):
    c = dict(CONFIGS[a.config])
    if a.tokens:
        c["T"] = a.tokens
    world = int(os.environ.get("WORLD_SIZE", a.gpus))
    c["etp_eff"] = c["etp"] if world >= 2 else 1
    c["ep_eff"] = max(1, world // c["etp_eff"])
    a.experts, a.topk, a.hidden, a.ffn = c["E"], c["k"], c["H"], c["F"]
    a.tokens = c["T"]
    a.cfg = c
    return c


def workload_config(a):
    c = a.cfg
    drop = "dropless" if c["cf"] is None else f"CF={c['cf']}" + (" pad-to-capacity" if c["pad"] else "")
    sh = f" + shared expert F={c['shared']}" if c["shared"] else ""
    return {"workload": f"{c['name']}: E{c['E']} top-{c['k']} H{c['H']} F{c['F']} SwiGLU{sh}, "
                        f"{c['T']} tokens/GPU, {drop}",
            "config": a.config, "tokens_per_gpu": c["T"], "experts": c["E"], "top_k": c["k"],
            "hidden": c["H"], "ffn": c["F"], "shared_ffn": c["shared"], "activation": "swiglu",
            "capacity_factor": c["cf"], "pad_to_capacity": c["pad"],
            "parallelism": f"ep{c['ep_eff']}" + (f"xetp{c['etp_eff']}" if c["etp_eff"] > 1 else ""),
            "l2": "per-step working set >10 GB (>> 126 MB L2); L2 also flushed between steps"}


# --------------------------------------------------------------- GPU arm
def relaunch(a) -> int:
    """`bench.py --gpus N` outside torchrun: re-run this script as N ranks
    (one process per GPU) under torch.distributed.run and return its code."""
    import socket
    import subprocess

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ and a.impl == "b200":
        sys.exit(relaunch(a))
    resolve(a)
    if a.impl == "reference":
        run_reference(a)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2504_14960_b200 as B
    from paper_2504_14960_b200 import _lib
    from paper_2504_14960_b200 import dispatcher as D
    from paper_2504_14960_b200 import gemm_tc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _lib.load()

    c = a.cfg
    E, k, H, F, T = c["E"], c["k"], c["H"], c["F"], c["T"]
    ep, etp = c["ep_eff"], c["etp_eff"]
    topo = B.ParallelTopology(world_size=world, ep=ep, etp=etp, tp=etp)
    seed = 0
    rng = np.random.default_rng([seed, 0])
    bnd = 1.0 / np.sqrt(H)
    wg = torch.as_tensor(rng.uniform(-bnd, bnd, size=(H, E)), dtype=torch.float32)
    params = B.GatingParams(w_g=wg, k=k, capacity_factor=c["cf"])
    L_ = E // ep
    etp_idx, ep_idx, _, _ = topo.moe_coords(rank)
    Fs = F // etp
    # random-init this rank's expert shards directly on the device (U(+-1/sqrt(H)))
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    w1 = [((torch.rand((H, 2 * Fs), generator=g, device=dev) * 2 - 1) * bnd) for _ in range(L_)]
    w2 = [((torch.rand((Fs, H), generator=g, device=dev) * 2 - 1) * bnd) for _ in range(L_)]
    weights = B.ExpertWeights(tuple(range(ep_idx * L_, (ep_idx + 1) * L_)), w1, w2, "swiglu",
                              etp_idx, etp)
    weights.packed(torch.bfloat16, dev)
    del w1, w2
    shared = None
    if c["shared"]:
        S_ = c["shared"]
        shared = B.ExpertWeights((0,), [(torch.rand((H, 2 * S_), generator=g, device=dev) * 2 - 1) * bnd],
                                 [(torch.rand((S_, H), generator=g, device=dev) * 2 - 1) * bnd],
                                 "swiglu", 0, 1)
        shared.packed(torch.bfloat16, dev)
    groups = B.generate_parallel_groups(topo)
    if world > 1:
        nw = B.NcclWorld()
        nw.setup_groups([groups.moe["EP"], groups.moe["ETP"], groups.moe["EDP"], [tuple(range(world))],
                         D.exchange_groups(topo)])
        ctx = B.collectives.NcclRankContext(nw)
    else:
        nw = B.LocalWorld(1, dev)
        ctx = B.collectives.LocalRankContext(nw, 0)
    layer = D.RankLayer(params, weights, topo, D._rank_groups(topo, groups, rank), rank,
                        torch.bfloat16, dev, shared=shared, pad_to_capacity=c["pad"])
    x = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
    u = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
    positions = torch.arange(T, dtype=torch.int64) + rank * T

    def step():
        out, sv = layer.forward(ctx, x, positions)
        dx, dwg, dw1, dw2 = layer.backward(ctx, u, sv)
        if world > 1:
            dwg = ctx.all_reduce(tuple(range(world)), dwg)
        return out, dx

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        step()
    barrier()
    if os.environ.get("B200MOE_NCU_RANGE") == "1":
        # exactly one step between cudaProfilerStart/Stop, for
        # `ncu --profile-from-start off` launch lists and captures
        torch.cuda.cudart().cudaProfilerStart()
        step()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        if world > 1:
            dist.destroy_process_group()
        return
    # ---- e2e through the public API with host (pinned) buffers: timed as
    # one run between the two halves of the resident-input steps, so both
    # legs see the same power/clock state (the GPU warms up over a run)
    run_e2e = None
    if not a.no_e2e and not a.profile_only:
        xh = x.cpu().pin_memory()
        uh = u.cpu().pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        dxh = torch.empty_like(xh).pin_memory()
        wmap = {(ep_idx, etp_idx): weights}
        api_world = nw
        from paper_2504_14960_b200.staging import HostStager

        stager = HostStager(dev)
        xd = [torch.empty_like(x), torch.empty_like(x)]  # double-buffered device tokens
        ud = torch.empty_like(u)
        state = {"x_ev": None}

        def e2e_step(i, last):
            # tokens for this step were uploaded during the previous step's
            # backward (or now, for the first step)
            if state["x_ev"] is None:
                state["x_ev"] = stager.upload(xh, xd[i % 2])
            u_ev = stager.upload(uh, ud)  # overlaps the forward
            stager.consume(state["x_ev"])
            blocks = [None] * world
            blocks[rank] = B.TokenBlock(xd[i % 2], positions)
            # the API's default path: inputs validated (router.py:141-144) through
            # the device status word, read after the router/dispatch barrier
            outs, fctx = B.moe_forward(blocks, wmap, topo, params, api_world, dtype=torch.bfloat16,
                                       shared_weights=shared, pad_to_capacity=c["pad"],
                                       check_finite_inputs=E2E_CHECK)
            stager.download(outs[rank], yh)  # overlaps the backward
            state["x_ev"] = None if last else stager.upload(xh, xd[(i + 1) % 2])
            stager.consume(u_ev)
            ups = [None] * world
            ups[rank] = ud
            res = B.moe_backward(ups, fctx)
            stager.download(res.input_grads[rank], dxh)  # overlaps the next forward

        def fresh_cache():
            # each leg starts from an empty caching allocator: blocks cached by
            # the other leg's tensor lifetimes (copy streams, per-call layers)
            # otherwise fragment the cache and the next leg's steps pay
            # cudaFree/cudaMalloc device syncs (C4 at 1 GPU: ~9 ms per step)
            barrier()
            torch.cuda.empty_cache()

        def run_e2e(n):
            """n pipelined API steps after one untimed one; ms for the n."""
            fresh_cache()
            e2e_step(0, True)
            stager.drain()
            barrier()
            m0 = torch.cuda.memory_stats()
            t0 = time.perf_counter()
            for i in range(n):
                e2e_step(i, i == n - 1)
            stager.drain()  # every step's copies complete inside the timed region
            barrier()
            t1 = time.perf_counter()
            if os.environ.get("B200MOE_BENCH_DEBUG") == "1":
                m1 = torch.cuda.memory_stats()
                print("e2e allocator:", {key: m1.get(key, 0) - m0.get(key, 0) for key in
                                         ("num_device_alloc", "num_device_free", "num_alloc_retries",
                                          "num_sync_all_streams")}, file=sys.stderr, flush=True)
            return (t1 - t0) * 1e3

        for i in range(2):
            e2e_step(i, i == 1)
        stager.drain()
        barrier()
    e2e_total_ms = 0.0
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)  # let the NVML poller start before the timed region
    total_ms = 0.0
    # every launch of the timed steps is bracketed by CUDA events on the
    # launching stream (the roofline's per-kernel durations come from these)
    per_step_launches = []
    launches = 0
    halves = [a.steps // 2, a.steps - a.steps // 2] if run_e2e is not None else [a.steps]
    t_wall0 = time.time()
    for hi, n_half in enumerate(halves):
        if hi or run_e2e is not None:
            if run_e2e is not None:
                fresh_cache()
            step()  # untimed: the resident-input path's buffers back in the allocator's cache
            barrier()
        _lib.reset_launch_count()
        for _ in range(n_half):
            flush.zero_()  # evict L2 between timed steps (outside the events)
            barrier()
            _lib.PROFILE.enable()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            barrier()
            per_step_launches.append(_lib.PROFILE.collect())
            _lib.PROFILE.disable()
            total_ms += e0.elapsed_time(e1)
        launches += _lib.launch_count()
        if run_e2e is not None and hi == 0:
            # all K e2e steps as one pipelined run between the two halves of
            # the resident-input steps: one exposed first upload / last
            # download per run, the same power/clock state as `value`
            e2e_total_ms += run_e2e(a.steps)
    t_wall1 = time.time()
    clocks.mark(t_wall0, t_wall1)
    clk = clocks.stop()
    ms = total_ms / a.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
    value = world * T / (ms / 1e3)
    e2e = None
    if run_e2e is not None:
        e2e_ms = e2e_total_ms / a.steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t)
        e2e = {"value": world * T / (e2e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 2 * xh.numel() * xh.element_size(),
               "d2h_bytes_per_step": 2 * yh.numel() * yh.element_size(),
               "ms_per_step": e2e_ms,
               "path": "moe_forward/moe_backward API (default: check_finite_inputs=True); pinned "
                       "host x/u in, y/dx out every step via HostStager copy streams overlapping compute; "
                       "timed as one pipelined run between the two halves of the resident-input steps"}

    # ---- roofline: expert GEMM launches averaged over the timed steps
    burst, sustained, hbm, src = peaks()
    nsteps = len(per_step_launches)
    n_launch = len(per_step_launches[0][0])
    all_launches = [(per_step_launches[0][0][i][0],
                     sum(s[0][i][1] for s in per_step_launches) / nsteps) for i in range(n_launch)]
    span_ms = sum(s[1] for s in per_step_launches) / nsteps
    per_launch = [(n, m) for n, m in all_launches if n.startswith("gemm_tc")]
    other = {}
    for n, m in all_launches:
        if not n.startswith("gemm_tc"):
            other[n] = other.get(n, 0.0) + m
    _, sv_last = layer.forward(ctx, x, positions)
    # all-to-all bus bandwidth (nccl-tests convention: bytes sent incl. self /
    # time * (n-1)/n), per direction per GPU, against 900 GB/s NVLink 5
    a2a = None
    a2a_events = [(n, m) for n, m in all_launches if n.startswith("nccl:a2a[")]
    if a2a_events and world > 1:
        sent = sum(int(n.split("[")[1].split("->")[0]) for n, _ in a2a_events) * H * 2
        t_a2a = sum(m for _, m in a2a_events) / 1e3
        busbw = sent / t_a2a * (world - 1) / world / 1e9
        a2a = {"busbw_gbs": busbw, "nominal_gbs": 900.0, "frac_nominal": busbw / 900.0,
               "ms_per_step": t_a2a * 1e3, "calls_per_step": len(a2a_events),
               "bytes_per_step": sent, "impl": "NCCL all_to_all_single (grouped P2P)"}
    peer_events = [(n, m) for n, m in all_launches if n == "ep_dispatch"]
    if peer_events and world > 1:
        # device-side exchange: the dispatch kernels push this rank's kept
        # rows to the etp members of each owning EP index, forward (x) and
        # backward (g*u); the rows that leave the GPU over the dispatch time is
        # the per-GPU, per-direction NVLink rate.  The return direction (y,
        # dx) is stored by the GEMM epilogues while they compute (no separate
        # time).  Exact bytes from the plan counts (peer.wire_rows semantics).
        from paper_2504_14960_b200.peer import wire_rows

        cnt = sv_last["plan_dev"].counts.to(torch.int64)
        _, e_idx, _, _ = topo.moe_coords(rank)
        per_ep = cnt.reshape(ep, -1).sum(1).cpu().tolist()
        pushed_rows = sum(c * (etp - (1 if j == e_idx else 0)) for j, c in enumerate(per_ep))
        px_last = sv_last.get("peer")
        dedup = bool(px_last is not None and px_last.dedup)
        if dedup:
            # one row per (token, remote EP index) crosses the link; rows for
            # this rank's own EP index stay per pair (also to its ETP
            # siblings, ep_peer.cu dispatch)
            dec = sv_last["dec"]
            dst = (dec.experts.to(torch.int64) // (E // ep)).masked_fill(~dec.kept.bool(), -1)
            per_dst = torch.stack([(dst == j).any(1).sum() for j in range(ep)]).cpu().tolist()
            pushed_rows = sum(c * etp for j, c in enumerate(per_dst) if j != e_idx) + \
                per_ep[e_idx] * (etp - 1)
        remote = 2 * pushed_rows * H * 2
        allc = [torch.empty_like(cnt) for _ in range(world)]
        dist.all_gather(allc, cnt)
        job_wire = wire_rows([c.reshape(ep, -1).cpu().numpy() for c in allc], topo) * H * 2
        t_x = sum(m for _, m in peer_events) / 1e3
        t_expand = sum(m for n_, m in all_launches if n_ == "ep_expand") / 1e3
        # launch order within a step: forward push (x), then backward push
        # (g*u, with the dgate dots against the returned rows)
        per_dir = {f"{d}_gbs": remote / 2 / (m / 1e3) / 1e9
                   for d, (_, m) in zip(("forward", "backward"), peer_events)} if len(peer_events) == 2 else None
        a2a = {"busbw_gbs": remote / t_x / 1e9, "nominal_gbs": 900.0,
               "frac_nominal": remote / t_x / 1e9 / 900.0,
               # measured peer-copy reference of this pool (B200_PROFILING.md): 770 GB/s per direction
               "measured_peer_gbs": 770.0, "frac_measured": remote / t_x / 1e9 / 770.0,
               "ms_per_step": t_x * 1e3, "expand_ms_per_step": t_expand * 1e3,
               "per_push": per_dir, "dedup": dedup,
               "remote_bytes_per_step": remote, "job_wire_bytes_per_step": job_wire,
               "impl": "NVLink peer memory: ep_dispatch push kernels + GEMM scatter epilogues (peer.py)"}
    # kept (token, expert) pairs of the last step, summed over ranks; each
    # pair costs 18*H*F flop fwd+bwd with SwiGLU (6PHF + 12PHF),
    # shared expert 18*T*H*Fs; per-GPU share of the whole job
    kept = torch.tensor([float(sv_last["plan_dev"].counts.sum())], device=dev)
    # rows this rank's expert GEMMs processed (pairs routed to its experts)
    if sv_last.get("pst") is not None:
        local_pairs = float(sv_last["pst"]["gcount"].sum())
    elif sv_last.get("xpl") is not None:
        # rows this member received; the ETP gather gives every member about etp x that
        local_pairs = float(sv_last["xpl"].recv_counts.sum()) * etp
    else:
        local_pairs = float(kept)
    gemm_ms = sum(ms_ for _, ms_ in per_launch)
    per_rank = None
    if world > 1:
        dist.all_reduce(kept)
        g = torch.tensor([local_pairs, gemm_ms], dtype=torch.float64, device=dev)
        allg = [torch.empty_like(g) for _ in range(world)]
        dist.all_gather(allg, g)
        per_rank = {"expert_rows": [int(v[0]) for v in allg],
                    "gemm_ms": [round(float(v[1]), 3) for v in allg]}
    P = local_pairs
    # each ETP member multiplies its rows by its F/etp shard
    flops_step = 18.0 * P * H * (F // etp) + 18.0 * T * H * c["shared"]
    achieved = flops_step / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
    roof = {"bound": "tensor", "kernel": "gemm_tc (grouped SwiGLU FFN, 6 launches/step)",
            "achieved": achieved, "peak": sustained, "unit": "TFLOP/s",
            "frac": achieved / sustained if achieved else None, "traffic": traffic(a.config),
            "peak_kind": f"{src} sustained bf16 (burst {burst})",
            "frac_of_burst": achieved / burst if achieved and burst else None,
            "frac_of_datasheet": achieved / 2250.0 if achieved else None,  # 2.25 PF dense bf16
            "algorithmic_flops_per_step": flops_step, "gemm_ms_per_step": gemm_ms,
            "gemm_share_of_step": gemm_ms / ms if ms else None,
            "launches_ms": [[n, round(m, 4)] for n, m in per_launch],
            "other_kernels_ms": {n: round(m, 4) for n, m in sorted(other.items(), key=lambda x: -x[1])},
            "instrumented_span_ms": span_ms,
            "launch_gaps_ms": span_ms - sum(m for _, m in all_launches),
            # the cross-GPU barriers in step order (time = wait for the slowest peer)
            "ep_barrier_ms": [round(m, 4) for n, m in all_launches if n == "ep_barrier"],
            "per_rank": per_rank,
            # whole layer: job tokens/s x average flop per token vs the per-GPU peak
            "layer_frac_of_peak": value / world * (18.0 * float(kept) / world * H * F / T
                                                   + 18.0 * H * c["shared"]) / 1e12 / sustained}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu and not a.profile_only:
        n = 256
        got = moefold_sample(a, 1, n, reps=3, warm=1)
        if got is not None:
            tok_s, threads, times, _ = got
            cpu = {"value": tok_s, "unit": UNIT, "cores": threads, "kind": "reference",
                   "source": "oracle/_ref/moefold",
                   "sample": f"{n} tokens, SimWorld(1), E{a.experts} top-{a.topk} H={a.hidden} "
                             f"F={a.ffn} ReLU (the reference has no SwiGLU), unmodified "
                             f"moefold.moe_forward+moe_backward, numpy float64, {threads} threads "
                             f"({cpu_model()}), mean of 3 reps after 1 warm-up"}
        else:
            tok_s, threads, _ = cpu_reference_sample(a, n, reps=3, warm=1)
            cpu = {"value": tok_s, "unit": UNIT, "cores": threads, "kind": "port",
                   "source": "oracle/moe_oracle.py",
                   "sample": f"{n} tokens at H={a.hidden} F={a.ffn} SwiGLU top-{a.topk}, numpy "
                             f"float64 oracle port of moe_forward+moe_backward, {threads} threads, "
                             f"mean of 3 reps after 1 warm-up"}

    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": workload_config(a),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "a2a": a2a,
            "gpu_launches": launches, "clocks": clk,
        }), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
