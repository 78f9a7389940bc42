"""Where does the e2e step time go?  (1 GPU, C2 shape)

    python tools/e2e_probe.py

(a) RankLayer forward+backward on device-resident tensors (bench `value`),
(b) moe_forward/moe_backward public API on device-resident tensors,
(c) (b) plus the pinned host copies of bench's e2e leg.
Each timed with CUDA events over a few steps after warm-up.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_14960_b200 as B  # noqa: E402
from paper_2504_14960_b200 import dispatcher as D  # noqa: E402
from paper_2504_14960_b200.staging import HostStager  # noqa: E402


def timed(fn, steps=4, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    t_host = (time.perf_counter() - t0) * 1e3 / steps
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, t_host


def main():
    E, k, H, F, T = 8, 2, 4096, 14336, int(os.environ.get("TOKENS", 16384))
    dev = torch.device("cuda", 0)
    topo = B.ParallelTopology(world_size=1)
    rng = np.random.default_rng([0, 0])
    bnd = 1.0 / np.sqrt(H)
    params = B.GatingParams(w_g=torch.as_tensor(rng.uniform(-bnd, bnd, size=(H, E)), dtype=torch.float32), k=k)
    g = torch.Generator(device=dev).manual_seed(1000)
    w1 = [((torch.rand((H, 2 * F), generator=g, device=dev) * 2 - 1) * bnd) for _ in range(E)]
    w2 = [((torch.rand((F, H), generator=g, device=dev) * 2 - 1) * bnd) for _ in range(E)]
    weights = B.ExpertWeights(tuple(range(E)), w1, w2, "swiglu", 0, 1)
    weights.packed(torch.bfloat16, dev)
    del w1, w2
    groups = B.generate_parallel_groups(topo)
    world = B.LocalWorld(1, dev)
    ctx = B.collectives.LocalRankContext(world, 0)
    layer = D.RankLayer(params, weights, topo, D._rank_groups(topo, groups, 0), 0, torch.bfloat16, dev)
    x = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
    u = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
    pos = torch.arange(T, dtype=torch.int64)

    def direct():
        _, sv = layer.forward(ctx, x, pos)
        layer.backward(ctx, u, sv)

    wmap = {(0, 0): weights}

    def api():
        outs, fctx = B.moe_forward([B.TokenBlock(x, pos)], wmap, topo, params, world, dtype=torch.bfloat16,
                                   check_finite_inputs=False)
        B.moe_backward([u], fctx)

    xh, uh = x.cpu().pin_memory(), u.cpu().pin_memory()
    yh, dxh = torch.empty_like(xh).pin_memory(), torch.empty_like(xh).pin_memory()
    st = HostStager(dev)
    xd, ud = torch.empty_like(x), torch.empty_like(u)

    def api_copies():
        ev = st.upload(xh, xd)
        ev2 = st.upload(uh, ud)
        st.consume(ev)
        outs, fctx = B.moe_forward([B.TokenBlock(xd, pos)], wmap, topo, params, world, dtype=torch.bfloat16,
                                   check_finite_inputs=False)
        st.download(outs[0], yh)
        st.consume(ev2)
        res = B.moe_backward([ud], fctx)
        st.download(res.input_grads[0], dxh)

    for name, fn in (("direct", direct), ("api", api), ("api+copies", api_copies)):
        ms, host = timed(fn)
        print(f"{name:12s} {ms:8.2f} ms/step (device)  {host:8.2f} ms/step (host enqueue)", flush=True)


if __name__ == "__main__":
    main()
