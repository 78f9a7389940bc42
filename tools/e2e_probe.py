"""Where does the e2e step time go?  (C2 shape; 1 GPU, or torchrun for EP = N)

    python tools/e2e_probe.py
    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/e2e_probe.py

(a) RankLayer forward+backward on device-resident tensors (bench `value`),
(b) moe_forward/moe_backward public API on device-resident tensors,
(c) (b) plus pinned host copies, serial (upload, step, download),
(d) (b) plus the copies pipelined across steps as in bench.py's e2e leg.
Each timed over a few steps after warm-up; wall-clock per step, max over ranks.
"""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_14960_b200 as B  # noqa: E402
from paper_2504_14960_b200 import dispatcher as D  # noqa: E402
from paper_2504_14960_b200.staging import HostStager  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    E, k, H, F, T = 8, 2, 4096, 14336, int(os.environ.get("TOKENS", 16384))
    steps = int(os.environ.get("STEPS", 6))
    topo = B.ParallelTopology(world_size=world, ep=world)
    rng = np.random.default_rng([0, 0])
    bnd = 1.0 / np.sqrt(H)
    params = B.GatingParams(w_g=torch.as_tensor(rng.uniform(-bnd, bnd, size=(H, E)), dtype=torch.float32), k=k)
    L_ = E // world
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    w1 = [((torch.rand((H, 2 * F), generator=g, device=dev) * 2 - 1) * bnd) for _ in range(L_)]
    w2 = [((torch.rand((F, H), generator=g, device=dev) * 2 - 1) * bnd) for _ in range(L_)]
    weights = B.ExpertWeights(tuple(range(rank * L_, (rank + 1) * L_)), w1, w2, "swiglu", 0, 1)
    weights.packed(torch.bfloat16, dev)
    del w1, w2
    groups = B.generate_parallel_groups(topo)
    if world > 1:
        nw = B.NcclWorld()
        nw.setup_groups([groups.moe["EP"], groups.moe["ETP"], groups.moe["EDP"], [tuple(range(world))],
                         D.exchange_groups(topo)])
        ctx = B.collectives.NcclRankContext(nw)
    else:
        nw = B.LocalWorld(1, dev)
        ctx = B.collectives.LocalRankContext(nw, 0)
    layer = D.RankLayer(params, weights, topo, D._rank_groups(topo, groups, rank), rank, torch.bfloat16, dev)
    x = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
    u = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
    pos = torch.arange(T, dtype=torch.int64) + rank * T
    wmap = {(rank, 0): weights}

    def sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, warm=2):
        for i in range(warm):
            fn(i, i == warm - 1)
        if hasattr(fn, "drain"):
            fn.drain()
        sync()
        t0 = time.perf_counter()
        host = 0.0
        for i in range(steps):
            h0 = time.perf_counter()
            fn(i, i == steps - 1)
            host += time.perf_counter() - h0
        if hasattr(fn, "drain"):
            fn.drain()
        sync()
        ms = (time.perf_counter() - t0) * 1e3 / steps
        t = torch.tensor([ms, host * 1e3 / steps], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0]), float(t[1])

    def direct(i, last):
        dwg = None
        _, sv = layer.forward(ctx, x, pos)
        _, dwg, _, _ = layer.backward(ctx, u, sv)
        if world > 1:
            ctx.all_reduce(tuple(range(world)), dwg)

    def blocks_of(v):
        b = [None] * world
        b[rank] = B.TokenBlock(v, pos)
        return b

    def ups_of(v):
        b = [None] * world
        b[rank] = v
        return b

    def api(i, last):
        if os.environ.get("ALLOC_STATS") == "1" and rank == 0:
            st_ = torch.cuda.memory_stats()
            print("alloc", {k_: st_.get(k_, 0) for k_ in ("num_device_alloc", "num_device_free",
                                                          "num_alloc_retries")}, flush=True)
        outs, fctx = B.moe_forward(blocks_of(x), wmap, topo, params, nw, dtype=torch.bfloat16,
                                   check_finite_inputs=False)
        B.moe_backward(ups_of(u), fctx)

    xh, uh = x.cpu().pin_memory(), u.cpu().pin_memory()
    yh, dxh = torch.empty_like(xh).pin_memory(), torch.empty_like(xh).pin_memory()
    st = HostStager(dev)
    xd = [torch.empty_like(x), torch.empty_like(x)]
    ud = torch.empty_like(u)

    def api_serial(i, last):
        ev = st.upload(xh, xd[0])
        ev2 = st.upload(uh, ud)
        st.consume(ev)
        outs, fctx = B.moe_forward(blocks_of(xd[0]), wmap, topo, params, nw, dtype=torch.bfloat16,
                                   check_finite_inputs=False)
        st.download(outs[rank], yh)
        st.consume(ev2)
        res = B.moe_backward(ups_of(ud), fctx)
        st.download(res.input_grads[rank], dxh)
        st.drain()

    state = {"x_ev": None}

    def api_pipelined(i, last):  # bench.py's e2e_step
        if state["x_ev"] is None:
            state["x_ev"] = st.upload(xh, xd[i % 2])
        u_ev = st.upload(uh, ud)
        st.consume(state["x_ev"])
        outs, fctx = B.moe_forward(blocks_of(xd[i % 2]), wmap, topo, params, nw, dtype=torch.bfloat16,
                                   check_finite_inputs=False)
        st.download(outs[rank], yh)
        state["x_ev"] = None if last else st.upload(xh, xd[(i + 1) % 2])
        st.consume(u_ev)
        res = B.moe_backward(ups_of(ud), fctx)
        st.download(res.input_grads[rank], dxh)

    api_pipelined.drain = st.drain
    which = os.environ.get("PROBES", "direct,api,serial,pipelined").split(",")
    for name, fn in (("direct", direct), ("api", api), ("api+copies serial", api_serial),
                     ("api+copies pipelined", api_pipelined)):
        if name.split()[-1] not in which:
            continue
        if os.environ.get("GAPS") == "1":
            # every rank runs the profiled steps (collectives); rank 0 reports
            import contextlib

            from torch.profiler import ProfilerActivity, profile

            for i in range(2):
                fn(i, False)
            sync()
            cm = profile(activities=[ProfilerActivity.CUDA]) if rank == 0 else contextlib.nullcontext()
            with cm as prof:
                for i in range(3):
                    fn(i, i == 2)
                if hasattr(fn, "drain"):
                    fn.drain()
                torch.cuda.synchronize()
            if rank != 0:
                ms, host = timed(fn)
                continue
            ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                        if e.device_type.name == "CUDA")
            gaps, end, prev = [], None, ""
            for s_, e_, n_ in ev:
                if end is not None and s_ - end > 50:
                    gaps.append((s_ - end, n_[:60] + "  (after " + prev[:40] + ")"))
                if end is None or e_ >= end:
                    prev = n_
                end = e_ if end is None else max(end, e_)
            busy = sum(e_ - s_ for s_, e_, _ in ev)
            print(f"{name}: span {(ev[-1][1] - ev[0][0]) / 1e3:.2f} ms, kernel sum {busy / 1e3:.2f} ms, "
                  f"gaps > 50 us: {len(gaps)} totalling {sum(g for g, _ in gaps) / 1e3:.2f} ms", flush=True)
            for g_, n_ in sorted(gaps, reverse=True)[:8]:
                print(f"   gap {g_:8.0f} us before {n_}", flush=True)
            per = {}
            for s_, e_, n_ in ev:
                key = n_[:48]
                c = per.setdefault(key, [0, 0.0])
                c[0] += 1
                c[1] += e_ - s_
            for key, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1])[:12]:
                print(f"   {c:4d} {t / 1e3:8.3f} ms  {key}", flush=True)
        if os.environ.get("PYPROF") == "1" and name == "api":  # every rank runs it (collectives)
            import cProfile
            import pstats

            timed(fn)  # first-use setup (exchange buffers, imports) outside the profile
            pr = cProfile.Profile()
            pr.enable()
            timed(fn)
            pr.disable()
            if rank == 0:
                pstats.Stats(pr).sort_stats("tottime").print_stats(22)
        ms, host = timed(fn)
        if rank == 0:
            print(f"{name:22s} {ms:8.2f} ms/step (wall, max over ranks)  {host:8.2f} ms/step host enqueue  "
                  f"{world * T / ms * 1e3:11.0f} tokens/s", flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
