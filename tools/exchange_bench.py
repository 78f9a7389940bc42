"""Time the peer-exchange push kernels alone (torchrun, >= 2 GPUs).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tools/exchange_bench.py [--tokens 16384] [--hidden 4096] [--topk 2] [--experts 8]

Routes random tokens, then times the forward push (ep_dispatch), the backward
push and the pair dots separately with CUDA events (barriers outside the
timed region) and prints the per-GPU, per-direction NVLink rate of each push
(remote bytes / kernel time) on rank 0.
"""
import argparse
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_14960_b200 as B  # noqa: E402
from paper_2504_14960_b200 import kernels as K  # noqa: E402
from paper_2504_14960_b200 import peer as PX  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--topk", type=int, default=2)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--hot", type=int, default=0,
                    help="bf16 8192^3 matmuls run right before each timed push (GPU in its "
                         "power-capped GEMM clock state, as inside a layer step)")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    T, H, k, E = a.tokens, a.hidden, a.topk, a.experts
    L_ = E // world
    g = torch.Generator(device=dev).manual_seed(rank)
    x = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
    logits = torch.randn((T, E), generator=g, device=dev)
    _, idx, gates, _ = K.router_topk(logits, k, 0, False)
    plan = K.dispatch_plan(idx, gates, E)
    nw = B.NcclWorld()
    ctx = B.collectives.NcclRankContext(nw)
    group = tuple(range(world))
    cap = PX.capacity_rows(world, T, k, L_, 128)
    ret = T * k + E * 127
    px = PX.PeerExchange(ctx, group, E, L_, H, cap, (ret + 127) // 128 * 128, dev)
    st = px.forward_dispatch(x, idx, plan, 128)
    y = px.region("yret")[0]
    per_ep = plan.counts.to(torch.int64).reshape(world, -1).sum(1).cpu().tolist()
    remote = sum(c for j, c in enumerate(per_ep) if j != rank) * H * 2

    hot_a = torch.randn((8192, 8192), device=dev).to(torch.bfloat16) if a.hot else None

    def timed(fn):
        ms = []
        for _ in range(a.reps):
            for _ in range(a.hot):
                hot_a @ hot_a
            px.barrier()
            if not a.hot:
                torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        ms.sort()
        return ms[len(ms) // 2]

    t_fwd = timed(lambda: K.ep_dispatch(x, idx, plan.gemm_row, plan.poffsets, st["seg_off"], L_,
                                        px.peer_base, px.me, 1, px.off["xr"], px.off["origin"]))
    t_bwd = timed(lambda: K.ep_dispatch(x, idx, plan.gemm_row, plan.poffsets, st["seg_off"], L_,
                                        px.peer_base, px.me, 1, px.off["dyr"], bwd=True, y_rows=y,
                                        gates=gates))
    if rank == 0:
        for name, t in (("fwd push", t_fwd), ("bwd push + dots", t_bwd)):
            print(f"{name:18s} {t * 1e3:8.1f} us   {remote / t / 1e6:7.1f} GB/s remote "
                  f"({remote / t / 1e6 / 900:5.1%} of 900)", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
