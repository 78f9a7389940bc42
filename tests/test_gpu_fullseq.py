"""GPU: full-sequence dropping on the device (router.py:209-269).

The group's pairs travel as int64 keys through a fixed-size all-gather, are
sorted on the device into admission order and one kernel applies the
per-sequence capacity (b200moe_fullseq_capacity): no host synchronisation,
no limit on sequences x experts.  Checked against the pinned oracle's
full_sequence_kept (which restates the reference's union / per-sequence
apply_capacity / map-back) and, for the layer, against the oracle's layer on
the GPU logits."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import moe_oracle as O  # noqa: E402

import paper_2504_14960_b200 as B  # noqa: E402
from paper_2504_14960_b200.errors import ProtocolError  # noqa: E402
from paper_2504_14960_b200.router import gather_full_sequence_decision  # noqa: E402

BF16_TOL = 2e-2


def t(a, dtype=torch.float32):
    return torch.as_tensor(np.asarray(a)).to("cuda", dtype).contiguous()


def _shards(rng, world, n_seq, seq_len, base):
    allpos = rng.permutation(n_seq * seq_len) + base * seq_len
    cuts = np.sort(rng.choice(np.arange(1, allpos.size), world - 1, replace=False))
    return np.split(allpos, cuts)


@pytest.mark.parametrize("priority", ["position", "probability"])
@pytest.mark.parametrize("E,k,seq_len,n_seq,world,cf", [(64, 8, 64, 100, 4, 1.0), (8, 2, 96, 5, 3, 1.0),
                                                        (16, 4, 128, 40, 2, 1.5)])
def test_device_full_sequence_capacity_vs_oracle(priority, E, k, seq_len, n_seq, world, cf):
    """Shuffled, ragged shards of many sequences (the first case has 6400
    sequence x expert segments, beyond the old 4096 limit); the layer-path
    call runs with torch's sync debug mode set to error: no host round trip."""
    rng = np.random.default_rng(E + n_seq)
    shards = _shards(rng, world, n_seq, seq_len, 3)
    params = B.GatingParams(w_g=np.eye(E), k=k, capacity_factor=cf, drop_mode="fullsequence",
                            drop_priority=priority)
    logits = [rng.standard_normal((s.size, E)).astype(np.float32) for s in shards]
    slots = max(s.size for s in shards)
    w = B.LocalWorld(world)
    decs = []
    for r in range(world):
        dec = B.router.routing_from_logits(t(logits[r]), params, shards[r])
        dec.positions = torch.as_tensor(shards[r]).cuda()  # device positions: no host copy in the call
        decs.append(dec)
    sts = [torch.zeros((1,), dtype=torch.int32, device="cuda") for _ in range(world)]
    torch.cuda.synchronize()

    def program(ctx):
        _, out = gather_full_sequence_decision(ctx, tuple(range(world)), decs[ctx.rank], seq_len, E, params,
                                               slots=slots, status=sts[ctx.rank], want_global=False)
        return decs[ctx.rank], out

    torch.cuda.set_sync_debug_mode("error")  # any synchronising CUDA call in the path raises
    try:
        res = w.run(program)
    finally:
        torch.cuda.set_sync_debug_mode("default")
    assert all(int(st) == 0 for st in sts)
    exps = [r[0].experts.cpu().numpy() for r in res]
    g64 = [r[0].gates_f64.cpu().numpy() if r[0].gates_f64 is not None else r[0].gates.double().cpu().numpy()
           for r in res]
    want = O.full_sequence_kept(exps, g64, shards, seq_len, cf, E, priority)
    for r in range(world):
        np.testing.assert_array_equal(res[r][1].kept.cpu().numpy(), want[r])


def test_global_decision_and_duplicate_positions():
    """The standalone API returns the group's union in position order with the
    capacity flags (router.py:236-262), and rejects duplicate positions."""
    E, k, seq_len, world = 8, 2, 64, 2
    rng = np.random.default_rng(5)
    shards = _shards(rng, world, 3, seq_len, 0)
    params = B.GatingParams(w_g=np.eye(E), k=k, capacity_factor=1.0, drop_mode="fullsequence")
    logits = [rng.standard_normal((s.size, E)).astype(np.float32) for s in shards]

    def program(ctx):
        dec = B.router.routing_from_logits(t(logits[ctx.rank]), params, shards[ctx.rank])
        return (dec,) + gather_full_sequence_decision(ctx, (0, 1), dec, seq_len, E, params)

    res = B.LocalWorld(world).run(program)
    exps = [r[0].experts.cpu().numpy() for r in res]
    g64 = [r[0].gates_f64.cpu().numpy() if r[0].gates_f64 is not None else r[0].gates.double().cpu().numpy()
           for r in res]
    want = O.full_sequence_kept(exps, g64, shards, seq_len, 1.0, E)
    pos = np.concatenate(shards)
    order = np.argsort(pos, kind="stable")
    glob = res[0][1]
    np.testing.assert_array_equal(glob.positions.numpy(), pos[order])
    np.testing.assert_array_equal(glob.experts.cpu().numpy(), np.concatenate(exps)[order])
    np.testing.assert_array_equal(glob.kept.cpu().numpy(), np.concatenate(want)[order])
    dup = [shards[0], np.concatenate([shards[1][:-1], shards[0][:1]])]

    def bad(ctx):
        dec = B.router.routing_from_logits(t(logits[ctx.rank]), params, dup[ctx.rank])
        gather_full_sequence_decision(ctx, (0, 1), dec, seq_len, E, params)

    with pytest.raises(ProtocolError, match="duplicate"):
        B.LocalWorld(world).run(bad)


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
def test_c5_like_full_sequence_layer_vs_oracle(exchange):
    """C5's mesh at reduced width: attention TP2 x CP2 over 4 ranks holding one
    16384-token sequence, MoE EP4, full-sequence dropping at CF 1.0, bf16:
    kept flags bit-exact and outputs within the bf16 tolerance of the oracle
    fed the GPU logits (identical-logit injection)."""
    E, k, H, F, seq_len, seed = 8, 2, 256, 512, 16384, 3
    topo = B.ParallelTopology(world_size=4, tp=2, cp=2, ep=4)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k, capacity_factor=1.0,
                            drop_mode="fullsequence")
    weights = B.init_expert_weights(E, H, F, 1, seed, ep_size=4, activation="swiglu")
    x_global, blocks = B.fabricate_token_blocks(topo, seq_len, topo.dp, H, seed, dtype=torch.bfloat16)
    outs, ctx = B.moe_forward(blocks, weights, topo, params, B.SimWorld(4), seq_len=seq_len,
                              exchange=exchange)
    torch.cuda.synchronize()
    positions = [b.positions.numpy() for b in blocks]
    lgs = [ctx.per_rank[r]["logits"].double().cpu().numpy() for r in range(4)]
    routs = [O.route_logits(lg, k) for lg in lgs]
    want = O.full_sequence_kept([r.experts for r in routs], [r.gates for r in routs], positions, seq_len,
                                1.0, E)
    full = B.init_expert_weights(E, H, F, 1, seed, activation="swiglu")[(0, 0)]
    experts = [O.Expert(np.asarray(a), np.asarray(b), "swiglu") for a, b in zip(full.w1, full.w2)]
    cfg = O.LayerConfig(k=k, capacity_factor=1.0)
    for r in range(4):
        np.testing.assert_array_equal(ctx.per_rank[r]["decision"].kept.cpu().numpy(), want[r])
        xr = blocks[r].values.float().cpu().numpy().astype(np.float64)
        yo, _ = O.layer_forward(xr, lgs[r], experts, cfg, positions=positions[r], kept_override=want[r])
        assert O.rel_err(outs[r].float().cpu().numpy(), yo) < BF16_TOL
    # the ledger charges the reference's width-4 routing gather over the sequence group
    recs = [rec for rec in ctx.world.ledger if rec.row_width == 4]
    assert len(recs) == 1 and recs[0].group == (0, 1, 2, 3)
    assert recs[0].elements_sent == tuple(4 * k * b.values.shape[0] * 3 for b in blocks)


def test_full_sequence_oversized_block_fails_every_rank():
    """A block larger than the gather slots agreed on first use fails the step
    on every rank through the status word (no rank leaves the collective)."""
    E, k, H, F, seq_len, seed = 8, 2, 64, 128, 256, 2
    topo = B.ParallelTopology(world_size=2, tp=2, ep=2)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k, capacity_factor=1.0,
                            drop_mode="fullsequence")
    weights = B.init_expert_weights(E, H, F, 1, seed, ep_size=2, activation="swiglu")
    world = B.LocalWorld(2)
    _, blocks = B.fabricate_token_blocks(topo, seq_len, topo.dp, H, seed, dtype=torch.bfloat16)
    _, ups = B.fabricate_upstream(topo, seq_len, topo.dp, H, seed, dtype=torch.bfloat16)
    _, c = B.moe_forward(blocks, weights, topo, params, world, seq_len=seq_len)
    B.moe_backward(ups, c)
    c.check()
    _, big = B.fabricate_token_blocks(topo, 2 * seq_len, topo.dp, H, seed, dtype=torch.bfloat16)
    _, bigu = B.fabricate_upstream(topo, 2 * seq_len, topo.dp, H, seed, dtype=torch.bfloat16)
    from paper_2504_14960_b200.errors import ValidationError

    with pytest.raises(ValidationError, match="first use"):
        _, c2 = B.moe_forward(big, weights, topo, params, world, seq_len=2 * seq_len)
        B.moe_backward(bigu, c2)
        c2.check()
