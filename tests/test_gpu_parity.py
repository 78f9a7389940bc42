"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the pinned CPU oracle.

Routing indices, kept masks, permutations and counts are compared bit-for-bit
given identical logits; floats within rel-err 1e-5 (fp32 mode) and 2e-2
(bf16) -- the tolerances of BASELINE.json's north star."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import moe_oracle as O  # noqa: E402

import paper_2504_14960_b200 as B  # noqa: E402
from paper_2504_14960_b200 import kernels as K  # noqa: E402

FP32_TOL = 1e-5
BF16_TOL = 2e-2


def _cases(d, prefix):
    return sorted({k.split("_")[0] for k in d if k.startswith(prefix)}, key=lambda s: int(s[1:]))


def t(a, dtype=torch.float32):
    return torch.as_tensor(np.asarray(a)).to("cuda", dtype).contiguous()


def test_library_loads_on_b200():
    from paper_2504_14960_b200 import _lib

    _lib.load()  # raises unless sm_100


def test_router_topk_matches_reference(golden):
    d = golden("router")
    for c in _cases(d, "r"):
        E, k, sig, renorm = (int(v) for v in d[c + "_meta"])
        scores, idx, gates, g64 = K.router_topk(t(d[c + "_logits"]), k, int(sig), bool(renorm), True)
        np.testing.assert_array_equal(idx.cpu().numpy(), d[c + "_experts"], err_msg=c)
        assert O.rel_err(g64.cpu().numpy(), d[c + "_gates"]) < 1e-14, c
        assert O.rel_err(gates.cpu().numpy(), d[c + "_gates"]) < 1e-6, c
        assert O.rel_err(scores.cpu().numpy(), d[c + "_scores"]) < 1e-6, c


def test_capacity_and_plan_match_reference(golden):
    d = golden("capacity_plan")
    for c in _cases(d, "c"):
        E, k, n, prob = (int(v) for v in d[c + "_meta"])
        cf = float(d[c + "_cf"][0])
        params = B.GatingParams(w_g=np.eye(E), k=k, capacity_factor=cf,
                                drop_priority="probability" if prob else "position")
        dec = B.router.routing_from_logits(t(d[c + "_logits"]), params)
        np.testing.assert_array_equal(dec.experts.cpu().numpy(), d[c + "_experts"])
        dropped = B.apply_capacity(dec, n, E, params)
        np.testing.assert_array_equal(dropped.kept.cpu().numpy(), d[c + "_kept"], err_msg=c)
        for ep in (1, 2, 4):
            if c + f"_perm_ep{ep}" not in d:
                continue
            plan = B.build_dispatch_plan(dropped, ep, E // ep)
            np.testing.assert_array_equal(plan.permutation, d[c + f"_perm_ep{ep}"], err_msg=c)
            np.testing.assert_array_equal(plan.send_counts, d[c + f"_counts_ep{ep}"], err_msg=c)
            assert O.rel_err(plan.gates, d[c + f"_pgates_ep{ep}"]) < 1e-6
        plan = B.build_dispatch_plan(dropped, 1, E)
        got = B.permute(t(d[c + "_x"]), plan).cpu().numpy()
        np.testing.assert_array_equal(got, d[c + "_permuted"].astype(np.float32))
        comb = B.unpermute_combine(t(d[c + "_rows"]), plan, 8).cpu().numpy()
        assert O.rel_err(comb, d[c + "_combined"]) < FP32_TOL, c


def test_plan_non_monotone_positions_and_edge_cases():
    rng = np.random.default_rng(3)
    E, k, n = 8, 2, 257
    logits = rng.standard_normal((n, E)).astype(np.float32)
    logits[:, 1] += 1.0
    positions = rng.permutation(n) + 1000
    params = B.GatingParams(w_g=np.eye(E), k=k, capacity_factor=1.0)
    dec = B.router.routing_from_logits(t(logits), params, positions)
    got = B.apply_capacity(dec, n, E, params).kept.cpu().numpy()
    r = O.route_logits(logits, k)
    want = O.apply_capacity(r.experts, r.gates, r.kept, positions, O.capacity_limit(1.0, n, E), E)
    np.testing.assert_array_equal(got, want)
    # empty block, single token, k == E
    for n_, k_ in ((0, 2), (1, 2), (5, 8)):
        lg = rng.standard_normal((n_, E)).astype(np.float32)
        p = B.GatingParams(w_g=np.eye(E), k=k_)
        dec = B.router.routing_from_logits(t(lg).reshape(n_, E), p)
        plan = B.build_dispatch_plan(dec, 2, 4)
        want = O.build_dispatch_plan(O.route_logits(lg.reshape(n_, E), k_).experts,
                                     np.ones((n_, k_)), np.ones((n_, k_), bool), 2, 4)
        np.testing.assert_array_equal(plan.permutation, want.permutation)
        np.testing.assert_array_equal(plan.send_counts, want.send_counts)


@pytest.mark.parametrize("dtype,tol", [(torch.float32, FP32_TOL), (torch.bfloat16, BF16_TOL)])
def test_expert_shards_match_reference(golden, dtype, tol):
    """fp32: against the reference's own outputs.  bf16: against the oracle
    evaluated on the same bf16-representable inputs and weights."""
    d = golden("experts")
    rnd = lambda a: t(a, dtype).double().cpu().numpy()  # noqa: E731
    for ci, act in enumerate(("relu", "gelu")):
        p = f"e{ci}_"
        w = B.ExpertWeights((0,), [d[p + "w1"]], [d[p + "w2"]], act, 0, 1)
        y, cache = B.expert_forward_shard(t(d[p + "x"], dtype), w, 0)
        dx, dw1, dw2 = B.expert_backward_shard(t(d[p + "u"], dtype), cache, w, 0)
        if dtype == torch.float32:
            want = {k: d[p + k] for k in ("y", "dx", "dw1", "dw2")}
        else:
            ex = O.Expert(rnd(d[p + "w1"]), rnd(d[p + "w2"]), act)
            yo, pre = O.expert_forward(rnd(d[p + "x"]), ex)
            g = O.expert_backward(rnd(d[p + "u"]), rnd(d[p + "x"]), pre, ex)
            want = dict(y=yo, dx=g[0], dw1=g[1], dw2=g[2])
        for name, got in (("y", y), ("dx", dx), ("dw1", dw1), ("dw2", dw2)):
            err = O.rel_err(got.float().cpu().numpy(), want[name])
            assert err < tol, (act, name, err)


def _gpu_logits_per_rank(ctx):
    return [sv["logits"].cpu().numpy().astype(np.float64) for sv in ctx.per_rank]


def _run_layer_case(d, c, dtype, act=None):
    meta = [int(v) for v in d[c + "_meta"]]
    w, tp, cp, ep, etp, E, k, H, F, seq, batch, seed, full, sig, renorm, gelu = meta
    cf = float(d[c + "_cf"][0])
    topo = B.ParallelTopology(world_size=w, tp=tp, cp=cp, ep=ep, etp=etp)
    params = B.GatingParams(w_g=d[c + "_wg"], k=k, gate_fn="sigmoid" if sig else "softmax",
                            renormalize_topk=bool(renorm), capacity_factor=None if cf < 0 else cf,
                            drop_mode="fullsequence" if full else "subsequence")
    weights = B.init_expert_weights(E, H, F, etp_size=etp, seed=seed, ep_size=ep,
                                    activation=act or ("gelu" if gelu else "relu"))
    x, u = d[c + "_x"], d[c + "_u"]
    positions = [d[c + f"_positions{r}"] for r in range(w)]
    blocks = [B.TokenBlock(t(x[p], dtype), p) for p in positions]
    world = B.SimWorld(w)
    outs, ctx = B.moe_forward(blocks, weights, topo, params, world, seq_len=seq)
    res = B.moe_backward([t(u[p], dtype) for p in positions], ctx)
    return meta, params, positions, outs, ctx, res


def _check_ledger(golden_ledgers, c, ctx):
    """The SimWorld wire ledger equals the reference's record for record
    (epoch, round, group, primitive, row width, elements per member)."""
    got = [[r.epoch, r.seq, list(r.group), r.primitive, r.row_width, list(r.elements_sent)]
           for r in ctx.world.ledger]
    assert got == golden_ledgers[c], c
    # recv_counts filled after the exchange (dispatcher.py:313-316): pairs sent == received
    w = len(ctx.per_rank)
    sent = sum(int(ctx.per_rank[r]["plan"].send_counts.sum()) for r in range(w))
    recv = sum(int(ctx.per_rank[r]["plan"].recv_counts.sum()) for r in range(w))
    assert sent == recv, c


def test_layer_cases_match_reference_fp32(golden, ledgers):
    """moe_forward/moe_backward (fp32 mode) on every golden topology, ranks
    simulated on one GPU, vs the reference's own outputs and gradients."""
    d = golden("layer")
    tol = FP32_TOL
    for c in _cases(d, "l"):
        meta, params, positions, outs, ctx, res = _run_layer_case(d, c, torch.float32)
        _check_ledger(ledgers, c, ctx)
        w, E, k = meta[0], meta[5], meta[6]
        x = d[c + "_x"]
        y = np.zeros_like(x)
        dx = np.zeros_like(x)
        for r, p in enumerate(positions):
            dec = ctx.per_rank[r]["decision"]
            lg = ctx.per_rank[r]["logits"].cpu().numpy()
            ro = O.route_logits(lg, k, params.gate_fn, params.renormalize_topk)
            np.testing.assert_array_equal(dec.experts.cpu().numpy(), ro.experts, err_msg=c)
            np.testing.assert_array_equal(dec.experts.cpu().numpy(), d[c + "_experts"][p], err_msg=c)
            np.testing.assert_array_equal(dec.kept.cpu().numpy(), d[c + "_kept"][p], err_msg=c)
            y[p] = outs[r].float().cpu().numpy()
            dx[p] = res.input_grads[r].float().cpu().numpy()
        assert O.rel_err(y, d[c + "_y"]) < tol, (c, O.rel_err(y, d[c + "_y"]))
        assert O.rel_err(dx, d[c + "_dx"]) < tol, (c, O.rel_err(dx, d[c + "_dx"]))
        assert O.rel_err(res.w_g_grad.cpu().numpy(), d[c + "_dwg"]) < tol, c
        ep, etp = meta[3], meta[4]
        local = E // ep
        for e in range(E):
            ei, le = e // local, e % local
            g1 = torch.cat([res.expert_grads[(ei, tt)][0][le] for tt in range(etp)], dim=1)
            g2 = torch.cat([res.expert_grads[(ei, tt)][1][le] for tt in range(etp)], dim=0)
            assert O.rel_err(g1.cpu().numpy(), d[c + "_dw1"][e]) < tol, (c, e)
            assert O.rel_err(g2.cpu().numpy(), d[c + "_dw2"][e]) < tol, (c, e)


def test_layer_cases_bf16_vs_oracle_with_gpu_logits(golden, ledgers):
    """bf16 mode on the golden topologies vs the pinned oracle fed the GPU's own
    logits and the bf16-rounded inputs (routing bit-exact, values 2e-2)."""
    d = golden("layer")
    for c in _cases(d, "l"):
        meta, params, positions, outs, ctx, res = _run_layer_case(d, c, torch.bfloat16, "gelu")
        _check_ledger(ledgers, c, ctx)
        w, E, k, seq, full = meta[0], meta[5], meta[6], meta[9], meta[12]
        cf = float(d[c + "_cf"][0])
        cfg = O.LayerConfig(k=k, gate_fn=params.gate_fn, renormalize=params.renormalize_topk,
                            capacity_factor=None if cf < 0 else cf)
        experts = [O.Expert(d[c + "_w1"][e], d[c + "_w2"][e], "gelu")
                   for e in range(E)]
        lgs = [ctx.per_rank[r]["logits"].cpu().numpy().astype(np.float64) for r in range(w)]
        kept_over = [None] * w
        if full and cfg.capacity_factor is not None:
            routs = [O.route_logits(lg, k, cfg.gate_fn, cfg.renormalize) for lg in lgs]
            kept_over = O.full_sequence_kept([r.experts for r in routs], [r.gates for r in routs],
                                             positions, seq, cfg.capacity_factor, E)
        rnd = lambda a: t(a, torch.bfloat16).float().cpu().numpy().astype(np.float64)  # noqa: E731
        x, u = d[c + "_x"], d[c + "_u"]
        y = np.zeros_like(x); yw = np.zeros_like(x); dx = np.zeros_like(x); dxw = np.zeros_like(x)
        dwg_w = np.zeros_like(d[c + "_wg"])
        dw1_w = [np.zeros_like(d[c + "_w1"][e]) for e in range(E)]
        dw2_w = [np.zeros_like(d[c + "_w2"][e]) for e in range(E)]
        for r, p in enumerate(positions):
            yo, st = O.layer_forward(rnd(x[p]), lgs[r], experts, cfg, positions=p,
                                     kept_override=kept_over[r])
            g = O.layer_backward(rnd(u[p]), st, experts, cfg, w_g=d[c + "_wg"])
            dec = ctx.per_rank[r]["decision"]
            np.testing.assert_array_equal(dec.experts.cpu().numpy(), st.routing.experts, err_msg=c)
            np.testing.assert_array_equal(dec.kept.cpu().numpy(), st.routing.kept, err_msg=c)
            y[p], yw[p] = outs[r].float().cpu().numpy(), yo
            dx[p], dxw[p] = res.input_grads[r].float().cpu().numpy(), g[0]
            # weight gradients summed over ranks (dispatcher.py:492-499)
            dwg_w += g[2]
            for e in range(E):
                dw1_w[e] += g[3][e]
                dw2_w[e] += g[4][e]
        assert O.rel_err(y, yw) < BF16_TOL, (c, O.rel_err(y, yw))
        assert O.rel_err(dx, dxw) < BF16_TOL, (c, O.rel_err(dx, dxw))
        assert O.rel_err(res.w_g_grad.cpu().numpy(), dwg_w) < BF16_TOL, c
        ep, etp = meta[3], meta[4]
        local = E // ep
        for e in range(E):
            ei, le = e // local, e % local
            g1 = torch.cat([res.expert_grads[(ei, tt)][0][le] for tt in range(etp)], dim=1).cpu().numpy()
            g2 = torch.cat([res.expert_grads[(ei, tt)][1][le] for tt in range(etp)], dim=0).cpu().numpy()
            assert O.rel_err(g1, dw1_w[e]) < BF16_TOL, (c, e, O.rel_err(g1, dw1_w[e]))
            assert O.rel_err(g2, dw2_w[e]) < BF16_TOL, (c, e, O.rel_err(g2, dw2_w[e]))




@pytest.mark.parametrize("act", ["relu", "swiglu"])
@pytest.mark.parametrize("dtype,tol", [(torch.float32, FP32_TOL), (torch.bfloat16, BF16_TOL)])
@pytest.mark.parametrize("cf", [None, 1.0])
def test_c1_shape_layer_vs_oracle(act, dtype, tol, cf):
    """C1 (BASELINE.json configs[0]): E8 top-2, H1024, F2816, T4096, EP=1."""
    E, k, H, F, T, seed = 8, 2, 1024, 2816, 4096, 0
    if act == "swiglu":
        F = 2816  # multiple of 32
    topo = B.ParallelTopology(world_size=1)
    wg = O.gating_matrix(H, E, seed)
    params = B.GatingParams(w_g=wg, k=k, capacity_factor=cf)
    weights = B.init_expert_weights(E, H, F, 1, seed, activation=act)
    x = O.token_rows(T, H, seed, 2)
    u = O.token_rows(T, H, seed, 3)
    block = B.TokenBlock(t(x, dtype), np.arange(T))
    outs, ctx = B.moe_forward([block], weights, topo, params, B.LocalWorld(1))
    res = B.moe_backward([t(u, dtype)], ctx)
    lg = ctx.per_rank[0]["logits"].cpu().numpy().astype(np.float64)
    w0 = weights[(0, 0)]
    experts = [O.Expert(np.asarray(a), np.asarray(b), act) for a, b in zip(w0.w1, w0.w2)]
    cfg = O.LayerConfig(k=k, capacity_factor=cf)
    xin = x if dtype == torch.float32 else t(x, dtype).float().cpu().numpy().astype(np.float64)
    uin = u if dtype == torch.float32 else t(u, dtype).float().cpu().numpy().astype(np.float64)
    y, st = O.layer_forward(xin, lg, experts, cfg)
    masks = None
    if act == "relu":
        # relu' as the GPU saw it (pre within rounding of 0 may flip sign)
        sv = ctx.per_rank[0]
        pre = sv["pre"].float().cpu().numpy()
        poff = sv["plan_dev"].poffsets.cpu().numpy()
        cnt = sv["plan_dev"].counts.cpu().numpy()
        masks = {e: pre[poff[e]:poff[e] + cnt[e]] > 0 for e in range(E)}
    g = O.layer_backward(uin, st, experts, cfg, w_g=wg, relu_masks=masks)
    dec = ctx.per_rank[0]["decision"]
    np.testing.assert_array_equal(dec.experts.cpu().numpy(), st.routing.experts)
    np.testing.assert_array_equal(dec.kept.cpu().numpy(), st.routing.kept)
    assert O.rel_err(outs[0].float().cpu().numpy(), y) < tol
    assert O.rel_err(res.input_grads[0].float().cpu().numpy(), g[0]) < tol
    assert O.rel_err(res.w_g_grad.cpu().numpy(), g[2]) < tol
    for e in range(E):
        assert O.rel_err(res.expert_grads[(0, 0)][0][e].cpu().numpy(), g[3][e]) < tol
        assert O.rel_err(res.expert_grads[(0, 0)][1][e].cpu().numpy(), g[4][e]) < tol


@pytest.mark.parametrize("dtype,tol", [(torch.float32, FP32_TOL), (torch.bfloat16, BF16_TOL)])
def test_c4_flavour_shared_expert_vs_oracle(dtype, tol):
    """C4 flavour (many experts, top-8, SwiGLU + dense shared expert; shapes
    reduced): routed + shared output and all gradients vs the oracle."""
    from paper_2504_14960_b200.experts import init_shared_expert

    E, k, H, F, Fs, T, seed = 64, 8, 256, 128, 512, 1024, 3
    wg = O.gating_matrix(H, E, seed)
    params = B.GatingParams(w_g=wg, k=k)
    weights = B.init_expert_weights(E, H, F, 1, seed, activation="swiglu")
    shared = init_shared_expert(H, Fs, seed)
    x = O.token_rows(T, H, seed, 2)
    u = O.token_rows(T, H, seed, 3)
    outs, ctx = B.moe_forward([B.TokenBlock(t(x, dtype), np.arange(T))], weights,
                              B.ParallelTopology(world_size=1), params, B.LocalWorld(1),
                              shared_weights=shared)
    res = B.moe_backward([t(u, dtype)], ctx)
    rnd = lambda a: t(a, dtype).double().cpu().numpy()  # noqa: E731
    lg = ctx.per_rank[0]["logits"].double().cpu().numpy()
    w0 = weights[(0, 0)]
    experts = [O.Expert(np.asarray(a), np.asarray(b), "swiglu") for a, b in zip(w0.w1, w0.w2)]
    sh = O.Expert(np.asarray(shared.w1[0]), np.asarray(shared.w2[0]), "swiglu")
    cfg = O.LayerConfig(k=k)
    y, st = O.layer_forward(rnd(x), lg, experts, cfg, shared=sh)
    g = O.layer_backward(rnd(u), st, experts, cfg, w_g=wg, shared=sh)
    np.testing.assert_array_equal(ctx.per_rank[0]["decision"].experts.cpu().numpy(), st.routing.experts)
    assert O.rel_err(outs[0].double().cpu().numpy(), y) < tol
    assert O.rel_err(res.input_grads[0].double().cpu().numpy(), g[0]) < tol
    assert O.rel_err(res.w_g_grad.cpu().numpy(), g[2]) < tol
    assert O.rel_err(res.shared_grads[0].cpu().numpy(), g[5][0]) < tol
    assert O.rel_err(res.shared_grads[1].cpu().numpy(), g[5][1]) < tol
    for e in range(0, E, 7):
        assert O.rel_err(res.expert_grads[(0, 0)][0][e].cpu().numpy(), g[3][e]) < tol


@pytest.mark.parametrize("world,ep,etp,tp", [(1, 1, 1, 1), (4, 2, 2, 2), (2, 2, 1, 1)])
def test_pad_to_capacity_equals_unpadded(world, ep, etp, tp):
    """C3 flavour: CF=1 dropping with pad-to-capacity (static segment sizes,
    no count exchange) gives the same outputs and gradients as the
    count-driven layout (no reference exists for padding; results must not
    change) -- fp32, emulated ranks."""
    E, k, H, F, seq, seed = 8, 2, 128, 256, 512, 21
    topo = B.ParallelTopology(world_size=world, tp=tp, ep=ep, etp=etp)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k, capacity_factor=1.0)
    weights = B.init_expert_weights(E, H, F, etp, seed, ep_size=ep, activation="swiglu")
    _, blocks = B.fabricate_token_blocks(topo, seq, topo.dp, H, seed)
    _, ups = B.fabricate_upstream(topo, seq, topo.dp, H, seed)
    runs = []
    for pad in (False, True):
        outs, ctx = B.moe_forward(blocks, weights, topo, params, B.LocalWorld(world), seq_len=seq,
                                  pad_to_capacity=pad)
        res = B.moe_backward(ups, ctx)
        runs.append((outs, res, ctx))
    (o0, r0, c0), (o1, r1, c1) = runs
    for r in range(world):
        np.testing.assert_array_equal(c0.per_rank[r]["decision"].kept.cpu().numpy(),
                                      c1.per_rank[r]["decision"].kept.cpu().numpy())
        assert c1.per_rank[r]["layer"].seg > 0
        assert O.rel_err(o1[r].cpu().numpy(), o0[r].cpu().numpy()) < 1e-6
        assert O.rel_err(r1.input_grads[r].cpu().numpy(), r0.input_grads[r].cpu().numpy()) < 1e-6
    assert O.rel_err(r1.w_g_grad.cpu().numpy(), r0.w_g_grad.cpu().numpy()) < 1e-6
    for key in r0.expert_grads:
        for a, b in zip(r0.expert_grads[key][0], r1.expert_grads[key][0]):
            assert O.rel_err(b.cpu().numpy(), a.cpu().numpy()) < 1e-6


@pytest.mark.parametrize("priority", ["position", "probability"])
def test_full_sequence_capacity_many_sequences_vs_oracle(priority):
    """Device full-sequence dropping (one virtual-expert capacity pass over all
    sequences of a group) vs the oracle: 3 ranks share a group holding 5
    sequences, positions shuffled and ragged across the shards."""
    from paper_2504_14960_b200.router import gather_full_sequence_decision

    E, k, seq_len, n_seq, world = 8, 2, 96, 5, 3
    rng = np.random.default_rng(11)
    allpos = rng.permutation(n_seq * seq_len) + 7 * seq_len  # sequences 7..11
    cuts = np.sort(rng.choice(np.arange(1, allpos.size), world - 1, replace=False))
    shards = np.split(allpos, cuts)
    params = B.GatingParams(w_g=np.eye(E), k=k, capacity_factor=1.0, drop_mode="fullsequence",
                            drop_priority=priority)
    logits = [rng.standard_normal((s.size, E)).astype(np.float32) for s in shards]
    world_ = B.LocalWorld(world)

    def program(ctx):
        r = ctx.rank
        dec = B.router.routing_from_logits(t(logits[r]), params, shards[r])
        _, out = gather_full_sequence_decision(ctx, tuple(range(world)), dec, seq_len, E, params)
        return dec, out

    res = world_.run(program)
    exps = [r[0].experts.cpu().numpy() for r in res]
    g64 = [r[0].gates_f64.cpu().numpy() if r[0].gates_f64 is not None else r[0].gates.double().cpu().numpy()
           for r in res]
    want = O.full_sequence_kept(exps, g64, shards, seq_len, 1.0, E, priority)
    for r in range(world):
        np.testing.assert_array_equal(res[r][1].kept.cpu().numpy(), want[r])


@pytest.mark.parametrize("E,k,n,gate", [(8, 2, 1000, "softmax"), (64, 8, 777, "sigmoid"), (4, 1, 0, "softmax")])
def test_load_stats_kernel_vs_oracle(E, k, n, gate):
    """router_stats kernel (load_stats, router.py:279-301) vs the oracle, with drops."""
    rng = np.random.default_rng(E + n)
    logits = rng.standard_normal((n, E)).astype(np.float32)
    params = B.GatingParams(w_g=np.eye(E), k=k, gate_fn=gate, capacity_factor=1.0)
    dec = B.router.routing_from_logits(t(logits).reshape(n, E), params)
    dec = B.apply_capacity(dec, n, E, params) if n else dec
    got = B.load_stats(dec, E)
    want = O.load_stats(dec.experts.cpu().numpy(), dec.kept.cpu().numpy(),
                        dec.scores.double().cpu().numpy(), E)
    np.testing.assert_array_equal(got.counts, want[0])
    if n:
        assert abs(got.imbalance - want[1]) < 1e-12
        assert abs(got.aux_loss - want[2]) < 1e-6 * max(1.0, abs(want[2]))


@pytest.mark.parametrize("gate_fn,renorm,priority", [("softmax", True, "probability"), ("sigmoid", False, "probability"),
                                                     ("sigmoid", True, "position")])
def test_bf16_layer_gating_variants_vs_oracle(gate_fn, renorm, priority):
    """bf16 layer through the fused tensor-core router (router_tc.cu) with the
    gating variants the golden layer cases do not cover: renormalised gates,
    sigmoid, probability-priority dropping (router.py:146-153, 195).  Kept
    masks equal the oracle's on the GPU logits; outputs and gradients within
    the bf16 tolerance."""
    E, k, H, F, T, seed = 8, 2, 512, 1024, 2048, 4
    topo = B.ParallelTopology(world_size=1)
    wg = O.gating_matrix(H, E, seed)
    params = B.GatingParams(w_g=wg, k=k, gate_fn=gate_fn, renormalize_topk=renorm, capacity_factor=1.0,
                            drop_priority=priority)
    weights = B.init_expert_weights(E, H, F, 1, seed, activation="swiglu")
    x = O.token_rows(T, H, seed, 2)
    u = O.token_rows(T, H, seed, 3)
    xb, ub = t(x, torch.bfloat16), t(u, torch.bfloat16)
    outs, ctx = B.moe_forward([B.TokenBlock(xb, np.arange(T))], weights, topo, params, B.LocalWorld(1))
    res = B.moe_backward([ub], ctx)
    ctx.check()
    lg = ctx.per_rank[0]["logits"].cpu().numpy().astype(np.float64)
    w0 = weights[(0, 0)]
    experts = [O.Expert(np.asarray(a), np.asarray(b), "swiglu") for a, b in zip(w0.w1, w0.w2)]
    cfg = O.LayerConfig(k=k, gate_fn=gate_fn, renormalize=renorm, capacity_factor=1.0, drop_priority=priority)
    xin = xb.float().cpu().numpy().astype(np.float64)
    uin = ub.float().cpu().numpy().astype(np.float64)
    y, st = O.layer_forward(xin, lg, experts, cfg)
    g = O.layer_backward(uin, st, experts, cfg, w_g=wg)
    dec = ctx.per_rank[0]["decision"]
    np.testing.assert_array_equal(dec.experts.cpu().numpy(), st.routing.experts)
    np.testing.assert_array_equal(dec.kept.cpu().numpy(), st.routing.kept)
    assert O.rel_err(outs[0].float().cpu().numpy(), y) < BF16_TOL
    assert O.rel_err(res.input_grads[0].float().cpu().numpy(), g[0]) < BF16_TOL
    assert O.rel_err(res.w_g_grad.cpu().numpy(), g[2]) < BF16_TOL
