"""NVLink bytes of the EP exchange, for ncu: the C2 layer (E8 top-2 H4096
F14336) on N GPUs as threads of ONE process (LocalWorld(devices=[...]), host
rendezvous barriers, so ncu's serialised kernel replay cannot deadlock a
device barrier), forward + backward once after a warm-up step.

Prints, per rank, the bytes the exchange must move over NVLink per launch
(from the plan counts: rows pushed to remote GPUs x H x 2, and rows the
scatter epilogue returns to remote GPUs), to compare with ncu's
nvltx__bytes / nvlrx__bytes of the ep_dispatch and gemm_tc launches:

  ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum \\
      -k regex:"ep_dispatch|gemm_tc" python tools/nvlink_probe.py --gpus 2
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_14960_b200 as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--topk", type=int, default=2)
    a = ap.parse_args()
    n, T, H, F, E, k = a.gpus, a.tokens, a.hidden, a.ffn, a.experts, a.topk
    os.environ.setdefault("B200MOE_PUSH_DEDUP", "0")
    topo = B.ParallelTopology(world_size=n, ep=n)
    rng = np.random.default_rng([0, 0])
    b = 1.0 / np.sqrt(H)
    params = B.GatingParams(w_g=rng.uniform(-b, b, size=(H, E)), k=k)
    L = E // n
    weights = {}
    for r in range(n):
        dev = torch.device("cuda", r)
        g = torch.Generator(device=dev).manual_seed(r)
        w1 = [((torch.rand((H, 2 * F), generator=g, device=dev) * 2 - 1) * b) for _ in range(L)]
        w2 = [((torch.rand((F, H), generator=g, device=dev) * 2 - 1) * b) for _ in range(L)]
        weights[(r, 0)] = B.ExpertWeights(tuple(range(r * L, (r + 1) * L)), w1, w2, "swiglu", 0, 1)
    blocks, ups = [], []
    for r in range(n):
        dev = torch.device("cuda", r)
        g = torch.Generator(device=dev).manual_seed(100 + r)
        blocks.append(B.TokenBlock(torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16),
                                   np.arange(r * T, (r + 1) * T)))
        ups.append(torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16))
    world = B.LocalWorld(n, devices=list(range(n)))
    for _ in range(2):
        outs, ctx = B.moe_forward(blocks, weights, topo, params, world, dtype=torch.bfloat16)
        B.moe_backward(ups, ctx)
    for r in range(n):
        torch.cuda.synchronize(r)
    rows = {}
    for r in range(n):
        plan = ctx.per_rank[r]["plan"]
        sent = plan.send_counts.sum(axis=1)  # rows to each EP rank (forward push)
        recv = plan.recv_counts.sum(axis=1)  # rows from each EP rank (returned by the scatter)
        rows[r] = {"push_rows_remote": int(sent.sum() - sent[r]),
                   "scatter_rows_remote": int(recv.sum() - recv[r])}
        rows[r]["push_bytes_remote"] = rows[r]["push_rows_remote"] * H * 2
        rows[r]["scatter_bytes_remote"] = rows[r]["scatter_rows_remote"] * H * 2
    print(json.dumps({"gpus": n, "tokens": T, "hidden": H, "per_rank": rows}))


if __name__ == "__main__":
    main()
