"""Multi-GPU parity check of the NCCL and NVLink peer-memory paths (run under torchrun, >= 2 GPUs).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port 29511 tests/dist_layer_check.py

Every rank runs moe_forward/moe_backward over NCCL (one process per GPU) and,
independently, the same topology with all ranks emulated on its own GPU
(LocalWorld), then compares its rank's outputs and gradients.  Also checks
the NCCL result against the CPU oracle fed the GPU logits.  Exits non-zero on
any mismatch."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2504_14960_b200 as B  # noqa: E402
from oracle import moe_oracle as O  # noqa: E402


def rel(a, b):
    a = a.double()
    b = b.double()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def cases(world):
    # tp, cp, ep, etp, cf, drop_mode, act, E, k -- the last case of each list
    # has top-4 with several experts per EP index: the deduplicated push runs
    # across GPUs (flag barrier, leader rows written over NVLink, ep_expand)
    if world == 2:
        return [(1, 1, 2, 1, None, "subsequence", "swiglu", 8, 2), (2, 1, 1, 2, None, "subsequence", "relu", 8, 2),
                (1, 2, 2, 1, 1.0, "fullsequence", "gelu", 8, 2), (2, 1, 2, 1, 1.0, "subsequence", "swiglu", 8, 2),
                (1, 1, 2, 1, None, "subsequence", "swiglu", 2, 2),  # one expert per rank (C2 at EP8)
                (1, 1, 2, 1, None, "subsequence", "swiglu", 16, 4)]
    return [(1, 1, world, 1, None, "subsequence", "swiglu", 8, 2), (2, 1, 2, 2, 1.0, "subsequence", "relu", 8, 2),
            (2, 2, 2, 2, 1.0, "fullsequence", "gelu", 8, 2),
            (1, 2, world // 2, 2, None, "subsequence", "swiglu", 8, 2),
            (1, 1, world, 1, None, "subsequence", "swiglu", world, 2),  # one expert per rank
            (1, 1, world, 1, None, "subsequence", "swiglu", 16, 4)]


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    H, F, seq = 128, 256, 256
    failures = []
    for ci, (tp, cp, ep, etp, cf, mode, act, E, k) in enumerate(cases(world)):
        for dtype, tol, xch in ((torch.float32, 1e-5, "nccl"), (torch.bfloat16, 2e-2, "peer"),
                                (torch.bfloat16, 2e-2, "nccl")):
            seed = 40 + ci
            topo = B.ParallelTopology(world_size=world, tp=tp, cp=cp, ep=ep, etp=etp)
            params = B.GatingParams(w_g=B.init_gating_matrix(H, E, seed), k=k, capacity_factor=cf,
                                    drop_mode=mode)
            weights = B.init_expert_weights(E, H, F, etp, seed, ep_size=ep, activation=act)
            _, blocks = B.fabricate_token_blocks(topo, seq, topo.dp, H, seed, dtype=dtype, device=dev)
            _, ups = B.fabricate_upstream(topo, seq, topo.dp, H, seed, dtype=dtype, device=dev)
            nw = B.NcclWorld()
            outs, fctx = B.moe_forward(blocks, weights, topo, params, nw, seq_len=seq, exchange=xch)
            res = B.moe_backward(ups, fctx)
            lw = B.LocalWorld(world, dev)
            outs2, fctx2 = B.moe_forward(blocks, weights, topo, params, lw, seq_len=seq, exchange=xch)
            res2 = B.moe_backward(ups, fctx2)
            torch.cuda.synchronize()
            peer = fctx.per_rank[rank].get("peer") is not None
            tag = f"case{ci} {topo} cf={cf} {mode} {act} {dtype} {'peer' if peer else 'nccl'}"
            d1 = fctx.per_rank[rank]["decision"]
            d2 = fctx2.per_rank[rank]["decision"]
            if not (torch.equal(d1.experts, d2.experts) and torch.equal(d1.kept, d2.kept)):
                failures.append(f"{tag}: routing differs")
            errs = {"y": rel(outs[rank], outs2[rank]), "dx": rel(res.input_grads[rank], res2.input_grads[rank]),
                    "dwg": rel(res.w_g_grad, res2.w_g_grad)}
            te, ee, de, pe = topo.moe_coords(rank)
            if de == 0:
                g1, g2 = res.expert_grads[(ee, te)], res2.expert_grads[(ee, te)]
                errs["dw1"] = max(rel(a, b) for a, b in zip(g1[0], g2[0]))
                errs["dw2"] = max(rel(a, b) for a, b in zip(g1[1], g2[1]))
            # against the oracle on the same (rounded) inputs with the GPU logits (no relu: smooth)
            if act != "relu" and mode == "subsequence":
                xin = blocks[rank].values.double().cpu().numpy()
                lg = fctx.per_rank[rank]["logits"].double().cpu().numpy()
                full = B.init_expert_weights(E, H, F, 1, seed, activation=act)[(0, 0)]
                exps = [O.Expert(np.asarray(a), np.asarray(b), act) for a, b in zip(full.w1, full.w2)]
                cfg = O.LayerConfig(k=k, capacity_factor=cf)
                yo, st = O.layer_forward(xin, lg, exps, cfg, positions=blocks[rank].positions.numpy())
                errs["y_vs_oracle"] = O.rel_err(outs[rank].double().cpu().numpy(), yo)
            worst = max(errs.values())
            status = "OK" if worst < tol else "FAIL"
            print(f"[rank {rank}] {status} {tag} " + " ".join(f"{n}={v:.2e}" for n, v in errs.items()),
                  flush=True)
            if worst >= tol:
                failures.append(tag)
            if peer and k >= 4:
                # the deduplicated push is bit-identical to the per-pair push
                # across GPUs (both settings agreed by every rank)
                assert fctx.per_rank[rank]["peer"].dedup
                os.environ["B200MOE_PUSH_DEDUP"] = "0"
                try:
                    outs0, fctx0 = B.moe_forward(blocks, weights, topo, params, nw, seq_len=seq, exchange=xch,
                                                 peer_tag="nodedup")
                    res0 = B.moe_backward(ups, fctx0)
                finally:
                    del os.environ["B200MOE_PUSH_DEDUP"]
                torch.cuda.synchronize()
                same = (torch.equal(outs0[rank], outs[rank]) and torch.equal(res0.input_grads[rank], res.input_grads[rank])
                        and torch.equal(res0.w_g_grad, res.w_g_grad) and not fctx0.per_rank[rank]["peer"].dedup)
                print(f"[rank {rank}] {'OK' if same else 'FAIL'} {tag} dedup push == per-pair push", flush=True)
                if not same:
                    failures.append(tag + " dedup")
    dist.barrier()
    dist.destroy_process_group()
    if failures:
        print(f"[rank {rank}] FAILURES: {failures}", flush=True)
        sys.exit(1)
    print(f"[rank {rank}] all multi-GPU parity checks passed", flush=True)


if __name__ == "__main__":
    main()
