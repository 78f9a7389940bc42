"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``moefold`` from /root/reference/pkg/src (read-only; no bytecode is
written) and stores inputs + reference outputs as compressed .npz fixtures
next to this script.  The fixtures travel with the repo; /root/reference does
not exist on the GPU box, so nothing at test time imports the reference.

Every router-level case feeds float32-representable logits through
``compute_gates(logits, GatingParams(w_g=eye(E), ...))`` which reproduces the
logits exactly, so the GPU path's float32 logits can be
checked against these decisions bit-for-bit.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from moefold import collectives as mc  # noqa: E402
from moefold import dispatcher as md  # noqa: E402
from moefold import experts as mx  # noqa: E402
from moefold import router as mr  # noqa: E402
from moefold.topology import ParallelTopology  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32_logits(rng, n, E, scale=2.0, tie_every=7):
    z = (rng.standard_normal((n, E)) * scale).astype(np.float32)
    # inject exact ties so the lower-id tie-break is exercised
    for i in range(0, n, tie_every):
        a, b = rng.choice(E, size=2, replace=False)
        z[i, b] = z[i, a]
    return z


def router_cases():
    rng = np.random.default_rng(20250421)
    out = {}
    cases = [
        (8, 2, "softmax", False), (8, 2, "softmax", True), (8, 1, "softmax", False),
        (8, 2, "sigmoid", False), (8, 2, "sigmoid", True), (64, 8, "softmax", False),
        (64, 8, "softmax", True), (64, 8, "sigmoid", False), (16, 4, "softmax", False),
        (4, 4, "softmax", True), (128, 8, "softmax", False), (32, 1, "sigmoid", False),
    ]
    for ci, (E, k, fn, renorm) in enumerate(cases):
        n = 160
        logits = f32_logits(rng, n, E)
        p = mr.GatingParams(w_g=np.eye(E), k=k, gate_fn=fn, renormalize_topk=renorm)
        dec = mr.compute_gates(logits.astype(np.float64), p)
        pre = f"r{ci}_"
        out[pre + "meta"] = np.array([E, k, fn == "sigmoid", renorm], dtype=np.int64)
        out[pre + "logits"] = logits
        out[pre + "experts"] = dec.experts
        out[pre + "gates"] = dec.gates
        out[pre + "scores"] = dec.scores
    return out


def capacity_cases():
    rng = np.random.default_rng(7)
    out = {}
    cases = [
        (8, 2, 1.0, "position", 512), (8, 2, 1.5, "position", 512), (8, 1, 1.0, "position", 333),
        (64, 8, 1.0, "position", 640), (64, 8, 2.0, "position", 640), (16, 4, 1.25, "position", 200),
        (8, 2, 1.0, "probability", 512), (64, 8, 1.0, "probability", 256), (4, 2, 1.0, "position", 7),
        (8, 2, 1.0, "position", 3),
    ]
    for ci, (E, k, cf, prio, n) in enumerate(cases):
        # skewed logits so capacity actually binds
        logits = f32_logits(rng, n, E, scale=1.0)
        logits[:, 0] += 1.5
        p = mr.GatingParams(w_g=np.eye(E), k=k, capacity_factor=cf, drop_priority=prio)
        dec = mr.compute_gates(logits.astype(np.float64), p)
        dropped = mr.apply_capacity(dec, n, E, p)
        pre = f"c{ci}_"
        out[pre + "meta"] = np.array([E, k, n, prio == "probability"], dtype=np.int64)
        out[pre + "cf"] = np.array([cf])
        out[pre + "logits"] = logits
        out[pre + "experts"] = dropped.experts
        out[pre + "gates"] = dropped.gates
        out[pre + "kept"] = dropped.kept
        out[pre + "cap"] = np.array([mr.capacity_limit(cf, n, E)])
        for ep in (1, 2, 4):
            if E % ep:
                continue
            plan = md.build_dispatch_plan(dropped, ep, E // ep)
            out[pre + f"perm_ep{ep}"] = plan.permutation
            out[pre + f"counts_ep{ep}"] = plan.send_counts
            out[pre + f"pgates_ep{ep}"] = plan.gates
        # permute / combine with the ep=1 plan
        plan = md.build_dispatch_plan(dropped, 1, E)
        x = rng.standard_normal((n, 8))
        rows = rng.standard_normal((plan.permutation.size, 8))
        out[pre + "x"] = x
        out[pre + "permuted"] = md.permute(x, plan)
        out[pre + "rows"] = rows
        out[pre + "combined"] = md.unpermute_combine(rows, plan, 8)
    return out


def expert_cases():
    rng = np.random.default_rng(11)
    out = {}
    for ci, act in enumerate(("relu", "gelu")):
        H, F, n = 24, 40, 33
        w1 = rng.standard_normal((H, F)) * 0.3
        w2 = rng.standard_normal((F, H)) * 0.3
        w = mx.ExpertWeights((0,), [w1], [w2], act, 0, 1)
        x = rng.standard_normal((n, H))
        u = rng.standard_normal((n, H))
        y, cache = mx.expert_forward_shard(x, w, 0)
        dx, dw1, dw2 = mx.expert_backward_shard(u, cache, w, 0)
        pre = f"e{ci}_"
        for name, v in dict(w1=w1, w2=w2, x=x, u=u, y=y, pre=cache[1], dx=dx, dw1=dw1, dw2=dw2).items():
            out[pre + name] = v
    return out


def layer_cases():
    """moe_forward / moe_backward on simulated worlds, small shapes."""
    out = {}
    cases = [
        # world, tp, cp, ep, etp, E, k, H, F, seq, cf, mode, fn, renorm, act
        (1, 1, 1, 1, 1, 8, 2, 32, 48, 64, None, "subsequence", "softmax", False, "relu"),
        (1, 1, 1, 1, 1, 8, 2, 32, 48, 64, 1.0, "subsequence", "softmax", False, "relu"),
        (1, 1, 1, 1, 1, 4, 2, 16, 24, 48, None, "subsequence", "sigmoid", True, "gelu"),
        (4, 2, 1, 2, 2, 4, 2, 16, 32, 32, None, "subsequence", "softmax", False, "relu"),
        (4, 1, 1, 4, 1, 8, 2, 16, 32, 32, 1.0, "subsequence", "softmax", True, "relu"),
        (4, 2, 2, 2, 2, 8, 2, 16, 32, 64, 1.0, "fullsequence", "softmax", False, "relu"),
        (4, 1, 2, 4, 1, 8, 2, 16, 32, 64, 1.0, "fullsequence", "sigmoid", False, "gelu"),
        (8, 2, 2, 4, 2, 8, 2, 16, 32, 64, 1.0, "subsequence", "softmax", False, "relu"),
    ]
    for ci, (w, tp, cp, ep, etp, E, k, H, F, seq, cf, mode, fn, renorm, act) in enumerate(cases):
        seed = 100 + ci
        topo = ParallelTopology(world_size=w, tp=tp, cp=cp, ep=ep, etp=etp)
        batch = topo.dp
        params = mr.GatingParams(
            w_g=mx.init_gating_matrix(H, E, seed), k=k, gate_fn=fn, renormalize_topk=renorm,
            capacity_factor=cf, drop_mode=mode,
        )
        weights = mx.init_expert_weights(E, H, F, etp_size=etp, seed=seed, ep_size=ep, activation=act)
        x_global, blocks = md.fabricate_token_blocks(topo, seq, batch, H, seed)
        world = mc.SimWorld(w)
        outs, ctx = md.moe_forward(blocks, weights, topo, params, world, seq_len=seq)
        u_global, ups = md.fabricate_upstream(topo, seq, batch, H, seed)
        res = md.moe_backward(ups, ctx)
        w1f, w2f = mx.full_expert_matrices(E, H, F, seed)
        pre = f"l{ci}_"
        out[pre + "meta"] = np.array([w, tp, cp, ep, etp, E, k, H, F, seq, batch, seed,
                                      mode == "fullsequence", fn == "sigmoid", renorm,
                                      act == "gelu"], dtype=np.int64)
        out[pre + "cf"] = np.array([-1.0 if cf is None else cf])
        out[pre + "x"] = x_global
        out[pre + "u"] = u_global
        out[pre + "wg"] = params.w_g
        out[pre + "w1"] = np.stack(w1f)
        out[pre + "w2"] = np.stack(w2f)
        y = np.zeros_like(x_global)
        dx = np.zeros_like(x_global)
        kept = np.zeros((x_global.shape[0], k), dtype=bool)
        experts = np.zeros((x_global.shape[0], k), dtype=np.int64)
        for r, b in enumerate(blocks):
            y[b.positions] = outs[r]
            dx[b.positions] = res.input_grads[r]
            kept[b.positions] = ctx.per_rank[r]["decision"].kept
            experts[b.positions] = ctx.per_rank[r]["decision"].experts
            out[pre + f"positions{r}"] = b.positions
            out[pre + f"perm{r}"] = ctx.per_rank[r]["plan"].permutation
            out[pre + f"counts{r}"] = ctx.per_rank[r]["plan"].send_counts
        out[pre + "y"] = y
        out[pre + "dx"] = dx
        out[pre + "kept"] = kept
        out[pre + "experts"] = experts
        out[pre + "dwg"] = res.w_g_grad
        # reassemble full expert grads from shards
        local = E // ep
        dw1 = np.zeros((E, H, F))
        dw2 = np.zeros((E, F, H))
        for e in range(E):
            ei, le = e // local, e % local
            dw1[e] = np.concatenate([res.expert_grads[(ei, t)][0][le] for t in range(etp)], axis=1)
            dw2[e] = np.concatenate([res.expert_grads[(ei, t)][1][le] for t in range(etp)], axis=0)
        out[pre + "dw1"] = dw1
        out[pre + "dw2"] = dw2
        # SimWorld wire ledger (collectives.py:11-18): token rows (width H) per
        # primitive; the full-sequence routing gather has width 4 and is skipped
        rows = {"all_to_all_v": 0, "all_gather_v": 0, "reduce_scatter_v": 0}
        for rec in world.ledger:
            if rec.primitive in rows and rec.row_width == H:
                rows[rec.primitive] += rec.total_elements // rec.row_width
        out[pre + "ledger_rows"] = np.array([rows["all_to_all_v"], rows["all_gather_v"],
                                             rows["reduce_scatter_v"]], dtype=np.int64)
        # the whole ledger, record by record (forward epoch 1, backward epoch 2)
        LEDGERS[pre.rstrip("_")] = [[rec.epoch, rec.seq, list(rec.group), rec.primitive, rec.row_width,
                                     list(rec.elements_sent)] for rec in world.ledger]
    return out


LEDGERS = {}


def topology_cases():
    from moefold.topology import LAYOUT_LISTING1, generate_parallel_groups, sequence_group
    import json

    out = []
    for w, tp, cp, pp, ep, etp, layout in [
        (8, 2, 2, 1, 8, 1, "pp-outermost"), (8, 2, 2, 1, 4, 2, "pp-outermost"),
        (16, 2, 4, 1, 8, 1, "pp-outermost"), (64, 2, 2, 2, 2, 2, "listing1"),
        (8, 2, 2, 2, 2, 1, "listing1"), (12, 3, 2, 2, 3, 2, "pp-outermost"),
    ]:
        topo = ParallelTopology(world_size=w, tp=tp, cp=cp, pp=pp, ep=ep, etp=etp, layout=layout)
        g = generate_parallel_groups(topo)
        out.append(dict(args=[w, tp, cp, pp, ep, etp, layout],
                        attention={k: [list(x) for x in v] for k, v in g.attention.items()},
                        moe={k: [list(x) for x in v] for k, v in g.moe.items()},
                        seq=[list(sequence_group(topo, r)) for r in range(w)],
                        attn_coords=[list(topo.attn_coords(r)) for r in range(w)],
                        moe_coords=[list(topo.moe_coords(r)) for r in range(w)]))
    for tp, cp, dp in [(2, 2, 2), (1, 2, 4), (2, 1, 1)]:
        topo = ParallelTopology(world_size=tp * cp * dp, tp=tp, cp=cp, ep=1)
        out.append(dict(partition=[tp, cp, dp],
                        parts=[p.tolist() for p in md.token_partition(topo, 16, 2 * dp)]))
    with open(os.path.join(OUT, "topology.json"), "w") as f:
        json.dump(out, f)


def main():
    topology_cases()
    np.savez_compressed(os.path.join(OUT, "router.npz"), **router_cases())
    np.savez_compressed(os.path.join(OUT, "capacity_plan.npz"), **capacity_cases())
    np.savez_compressed(os.path.join(OUT, "experts.npz"), **expert_cases())
    np.savez_compressed(os.path.join(OUT, "layer.npz"), **layer_cases())
    import json

    with open(os.path.join(OUT, "ledger.json"), "w") as f:
        json.dump(LEDGERS, f)
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
