"""Push beside a GEMM: rate of the side push (b200moe_ep_dispatch_part 2)
alone and concurrent with a persistent gemm_tc launch on another stream
(torchrun, 2+ GPUs, C2 shape by default).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/push_overlap_probe.py
"""
import argparse
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_14960_b200 as B  # noqa: E402
from paper_2504_14960_b200 import experts as X  # noqa: E402
from paper_2504_14960_b200 import gemm_tc  # noqa: E402
from paper_2504_14960_b200 import kernels as K  # noqa: E402
from paper_2504_14960_b200 import peer as PX  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    ap.add_argument("--topk", type=int, default=2)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    T, H, F, k, E = a.tokens, a.hidden, a.ffn, a.topk, a.experts
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
    st = px.forward_dispatch(x, idx, plan, 128, overlap=True)
    px.land(st)
    per_ep = plan.counts.to(torch.int64).reshape(world, -1).sum(1).cpu().tolist()
    remote = sum(c for j, c in enumerate(per_ep) if j != rank) * H * 2
    w1 = [torch.randn((H, 2 * F), device=dev) * 0.02 for _ in range(L_)]
    w2 = [torch.randn((F, H), device=dev) * 0.02 for _ in range(L_)]
    pk = B.ExpertWeights(tuple(range(L_)), w1, w2, "swiglu", 0, 1).packed(torch.bfloat16, dev)
    xr = px.region("xr")
    pre = torch.empty((cap, 2 * F), dtype=torch.bfloat16, device=dev)
    h = torch.empty((cap, F), dtype=torch.bfloat16, device=dev)
    side = torch.cuda.Stream(device=dev)
    args = (x, idx, plan.gemm_row, plan.poffsets, st["seg_off"], L_, px.peer_base, px.me, 1, px.off["xr"],
            px.off["origin"])

    def gemm():
        gemm_tc.ffn1_fused(xr, pk, pre, h, st["goff"], L_, None, cap)

    def push(part):
        K.ep_dispatch(*args, part=part)

    def run(fn_main, fn_side, gemm_first=False):
        res = []
        for _ in range(a.reps):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1, s0, s1 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
            side.wait_stream(torch.cuda.current_stream())

            def do_side():
                if fn_side:
                    with torch.cuda.stream(side):
                        s0.record()
                        fn_side()
                        s1.record()
            if not gemm_first:
                do_side()
            e0.record()
            if fn_main:
                fn_main()
            e1.record()
            if gemm_first:
                do_side()
            torch.cuda.synchronize()
            res.append((e0.elapsed_time(e1) if fn_main else 0.0, s0.elapsed_time(s1) if fn_side else 0.0))
        res.sort()
        return res[len(res) // 2]

    out = {}
    out["push0 alone"] = run(None, lambda: push(0))
    out["push2 alone"] = run(None, lambda: push(2))
    out["gemm alone"] = run(gemm, None)
    out["gemm + push2 (push first)"] = run(gemm, lambda: push(2))
    out["gemm + push0 (push first)"] = run(gemm, lambda: push(0))
    out["gemm + push2 (gemm first)"] = run(gemm, lambda: push(2), gemm_first=True)

    # the fair comparison: one region from a common idle start to both done
    def region(kind):
        res = []
        for _ in range(a.reps):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if kind == "serial":
                push(0)
                gemm()
            else:
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    push(2)
                gemm()
                torch.cuda.current_stream().wait_stream(side)
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1))
        res.sort()
        return res[len(res) // 2], 0.0

    out["serial push0 -> gemm (region)"] = region("serial")
    out["push2 beside gemm (region)"] = region("overlap")
    if rank == 0:
        bpsm = os.environ.get("B200MOE_PUSH_BLOCKS_PER_SM", "1") + " carve " + \
            os.environ.get("B200MOE_PUSH_CARVEOUT", "1")
        for name, (tg, tp) in out.items():
            rate = f"{remote / (tp * 1e-3) / 1e9:7.1f} GB/s" if tp else ""
            print(f"[blocks/SM {bpsm}] {name:28s} gemm {tg:8.3f} ms  push {tp:8.3f} ms {rate}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
