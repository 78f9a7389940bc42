"""GPU: the device-side EP exchange over peer memory (peer.py, csrc/ep_peer.cu)
against the NCCL-style exchange and the oracle.

Ranks are threads on one GPU (LocalWorld): the same dispatch / combine /
layout kernels run, with a host rendezvous in place of the flag barrier
(which tests/dist_layer_check.py exercises across real GPUs).  Expert rows
are computed by the same GEMM whatever their position in the receive buffer,
so forward outputs must match the NCCL path bit for bit; gradients differ
only in fp32 summation order."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import moe_oracle as O  # noqa: E402

import paper_2504_14960_b200 as B  # noqa: E402
from paper_2504_14960_b200.errors import ProtocolError, ValidationError  # noqa: E402

BF16_TOL = 2e-2


def _blocks(sizes, H, seed):
    rng = np.random.default_rng(seed)
    out, ups, start = [], [], 0
    for n in sizes:
        pos = np.arange(start, start + n)
        start += n
        out.append(B.TokenBlock(torch.as_tensor(rng.standard_normal((n, H)), dtype=torch.float32)
                                .to("cuda", torch.bfloat16), pos))
        ups.append(torch.as_tensor(rng.standard_normal((n, H)), dtype=torch.float32)
                   .to("cuda", torch.bfloat16))
    return out, ups


def _run(exchange, topo, params, weights, blocks, ups, shared=None):
    world = B.LocalWorld(topo.world_size)
    outs, ctx = B.moe_forward(blocks, weights, topo, params, world, dtype=torch.bfloat16,
                              exchange=exchange, shared_weights=shared)
    res = B.moe_backward(ups, ctx)
    return outs, ctx, res


CASES = [
    # world, ep, etp, E, k, H, F, sizes, cf, act
    (2, 2, 1, 8, 2, 256, 512, (384, 384), None, "swiglu"),
    (2, 2, 1, 8, 2, 128, 256, (96, 300), 1.0, "swiglu"),  # ragged blocks, dropping
    (4, 4, 1, 4, 2, 128, 192, (64, 128, 0, 200), None, "gelu"),  # k > L, an empty rank
    (4, 2, 1, 8, 4, 64, 128, (160, 96, 128, 64), 1.25, "swiglu"),  # ep < world (EDP = 2)
    (4, 4, 1, 16, 8, 64, 64, (256, 256, 256, 256), None, "swiglu"),  # k = 8
    (8, 8, 1, 8, 2, 128, 128, (128,) * 8, None, "swiglu"),  # the 8-GPU layout: one expert per rank
    (4, 2, 2, 8, 2, 128, 256, (192, 64, 128, 256), 1.0, "swiglu"),  # EP x ETP (C3 shape)
    (2, 1, 2, 4, 2, 64, 128, (100, 200), None, "swiglu"),  # ETP only
    (8, 2, 4, 8, 2, 64, 256, (64, 96, 32, 128, 64, 64, 80, 16), None, "gelu"),  # ETP 4
]


@pytest.mark.parametrize("world,ep,etp,E,k,H,F,sizes,cf,act", CASES)
def test_peer_exchange_matches_nccl_exchange(world, ep, etp, E, k, H, F, sizes, cf, act):
    seed = 11
    topo = B.ParallelTopology(world_size=world, ep=ep, etp=etp, tp=etp)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k, capacity_factor=cf)
    weights = B.init_expert_weights(E, H, F, etp, seed, ep_size=ep, activation=act)
    blocks, ups = _blocks(sizes, H, seed)
    o0, c0, r0 = _run("nccl", topo, params, weights, blocks, ups)
    o1, c1, r1 = _run("peer", topo, params, weights, blocks, ups)
    for r in range(world):
        assert c1.per_rank[r].get("peer") is not None
        assert c0.per_rank[r].get("peer") is None
        np.testing.assert_array_equal(c0.per_rank[r]["decision"].kept.cpu().numpy(),
                                      c1.per_rank[r]["decision"].kept.cpu().numpy())
        if sizes[r]:
            torch.testing.assert_close(o1[r], o0[r], rtol=0, atol=0)
            assert O.rel_err(r1.input_grads[r].float().cpu().numpy(),
                             r0.input_grads[r].float().cpu().numpy()) < 1e-2
    assert O.rel_err(r1.w_g_grad.cpu().numpy(), r0.w_g_grad.cpu().numpy()) < 1e-3
    for key in r0.expert_grads:
        for a, b in zip(r0.expert_grads[key][0] + r0.expert_grads[key][1],
                        r1.expert_grads[key][0] + r1.expert_grads[key][1]):
            assert O.rel_err(b.cpu().numpy(), a.cpu().numpy()) < 1e-3


def test_peer_exchange_with_shared_expert_vs_oracle():
    """2 emulated ranks, E16 top-4 SwiGLU + shared expert, bf16, vs the oracle
    fed the GPU's logits and bf16-rounded inputs."""
    from paper_2504_14960_b200.experts import init_shared_expert

    E, k, H, F, Fs, seed = 16, 4, 256, 256, 512, 5
    sizes = (512, 320)
    topo = B.ParallelTopology(world_size=2, ep=2)
    wg = O.gating_matrix(H, E, seed)
    params = B.GatingParams(w_g=wg, k=k)
    weights = B.init_expert_weights(E, H, F, 1, seed, ep_size=2, activation="swiglu")
    shared = init_shared_expert(H, Fs, seed)
    blocks, ups = _blocks(sizes, H, seed)
    outs, ctx, res = _run("peer", topo, params, weights, blocks, ups, shared)
    experts = []
    for ei in range(2):
        w = weights[(ei, 0)]
        experts += [O.Expert(np.asarray(a), np.asarray(b), "swiglu") for a, b in zip(w.w1, w.w2)]
    sh = O.Expert(np.asarray(shared.w1[0]), np.asarray(shared.w2[0]), "swiglu")
    cfg = O.LayerConfig(k=k)
    dwg = np.zeros_like(wg)
    for r in range(2):
        assert ctx.per_rank[r].get("peer") is not None
        lg = ctx.per_rank[r]["logits"].double().cpu().numpy()
        x = blocks[r].values.double().cpu().numpy()
        u = ups[r].double().cpu().numpy()
        y, st = O.layer_forward(x, lg, experts, cfg, shared=sh)
        g = O.layer_backward(u, st, experts, cfg, w_g=wg, shared=sh)
        np.testing.assert_array_equal(ctx.per_rank[r]["decision"].experts.cpu().numpy(),
                                      st.routing.experts)
        assert O.rel_err(outs[r].double().cpu().numpy(), y) < BF16_TOL
        assert O.rel_err(res.input_grads[r].double().cpu().numpy(), g[0]) < BF16_TOL
        dwg += g[2]
    assert O.rel_err(res.w_g_grad.cpu().numpy(), dwg) < BF16_TOL


def test_peer_buffers_reused_before_backward_fail_loudly():
    E, k, H, F = 8, 2, 64, 64
    topo = B.ParallelTopology(world_size=2, ep=2)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, 1), k=k)
    weights = B.init_expert_weights(E, H, F, 1, 1, ep_size=2, activation="swiglu")
    blocks, ups = _blocks((64, 64), H, 1)
    world = B.LocalWorld(2)
    _, ctx_a = B.moe_forward(blocks, weights, topo, params, world, dtype=torch.bfloat16)
    _, ctx_b = B.moe_forward(blocks, weights, topo, params, world, dtype=torch.bfloat16)
    B.moe_backward(ups, ctx_b)
    with pytest.raises(ProtocolError, match="reused"):
        B.moe_backward(ups, ctx_a)
    # a later, larger token block than the buffers were sized for
    big, _ = _blocks((128, 64), H, 2)
    with pytest.raises(ValidationError, match="peer buffers"):  # from moe_forward, moe_backward or check()
        _, ctx_big = B.moe_forward(big, weights, topo, params, world, dtype=torch.bfloat16)
        B.moe_backward(_blocks((128, 64), H, 3)[1], ctx_big)
        ctx_big.check()


def test_peer_tags_and_headroom():
    """Interleaved layers (fwd A, fwd B, bwd A, bwd B) on distinct peer tags
    give the results of running them one after the other, and buffers sized
    with ``peer_tokens`` accept a later, larger token block."""
    E, k, H, F = 8, 2, 64, 64
    topo = B.ParallelTopology(world_size=2, ep=2)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, 1), k=k)
    weights = B.init_expert_weights(E, H, F, 1, 1, ep_size=2, activation="swiglu")
    blocks, ups = _blocks((64, 96), H, 1)
    world = B.LocalWorld(2)
    o_ref, c_ref = B.moe_forward(blocks, weights, topo, params, world, dtype=torch.bfloat16)
    r_ref = B.moe_backward(ups, c_ref)
    world = B.LocalWorld(2)
    o_a, c_a = B.moe_forward(blocks, weights, topo, params, world, dtype=torch.bfloat16, peer_tag="a")
    o_b, c_b = B.moe_forward(blocks, weights, topo, params, world, dtype=torch.bfloat16, peer_tag="b")
    r_a = B.moe_backward(ups, c_a)
    r_b = B.moe_backward(ups, c_b)
    for r in range(2):
        for o in (o_a, o_b):
            torch.testing.assert_close(o[r], o_ref[r], rtol=0, atol=0)
        for res in (r_a, r_b):
            torch.testing.assert_close(res.input_grads[r], r_ref.input_grads[r], rtol=0, atol=0)
    world = B.LocalWorld(2)
    B.moe_forward(blocks, weights, topo, params, world, dtype=torch.bfloat16, peer_tokens=256)
    big, ups_big = _blocks((256, 200), H, 2)
    outs, ctx = B.moe_forward(big, weights, topo, params, world, dtype=torch.bfloat16)
    res = B.moe_backward(ups_big, ctx)
    o_n, c_n = B.moe_forward(big, weights, topo, params, B.LocalWorld(2), dtype=torch.bfloat16,
                             exchange="nccl")
    for r in range(2):
        torch.testing.assert_close(outs[r], o_n[r], rtol=0, atol=0)
    assert res.input_grads[0].shape == (256, H)


@pytest.mark.parametrize("ep,etp", [(2, 2), (4, 1)])
def test_peer_exchange_pad_to_capacity_matches_nccl(ep, etp):
    """C3 flavour on the device exchange: CF = 1 with pad-to-capacity segments
    (static local layout) against the NCCL path."""
    world, E, k, H, F, seed = 4, 8, 2, 128, 256, 13
    topo = B.ParallelTopology(world_size=world, ep=ep, etp=etp, tp=etp)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k, capacity_factor=1.0)
    weights = B.init_expert_weights(E, H, F, etp, seed, ep_size=ep, activation="swiglu")
    blocks, ups = _blocks((256, 256, 256, 256), H, seed)
    runs = []
    for xch in ("nccl", "peer"):
        wld = B.LocalWorld(world)
        outs, ctx = B.moe_forward(blocks, weights, topo, params, wld, dtype=torch.bfloat16,
                                  exchange=xch, pad_to_capacity=True)
        res = B.moe_backward(ups, ctx)
        assert all(ctx.per_rank[r]["layer"].seg > 0 for r in range(world))
        runs.append((outs, res))
    (o0, r0), (o1, r1) = runs
    for r in range(world):
        torch.testing.assert_close(o1[r], o0[r], rtol=0, atol=0)
        assert O.rel_err(r1.input_grads[r].float().cpu().numpy(),
                         r0.input_grads[r].float().cpu().numpy()) < 1e-2
    for key in r0.expert_grads:
        for a, b in zip(r0.expert_grads[key][0], r1.expert_grads[key][0]):
            assert O.rel_err(b.cpu().numpy(), a.cpu().numpy()) < 1e-3


_ABSENT_PEER = """
import torch
from paper_2504_14960_b200 import kernels as K
buf = torch.zeros(4096, dtype=torch.uint8, device="cuda")
base = torch.tensor([buf.data_ptr(), buf.data_ptr()], dtype=torch.int64, device="cuda")
K.ep_barrier(base, 0, 0, 2, 1)  # rank 1 never announces epoch 1
torch.cuda.synchronize()
print("NO TRAP")
"""


def test_barrier_with_an_absent_peer_traps_instead_of_hanging():
    """A member that never reaches the flag barrier makes the waiting rank
    trap after $B200MOE_BARRIER_TIMEOUT_S (a launch failure the host sees)
    rather than spin forever (run in a subprocess: the trap poisons the
    CUDA context)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, B200MOE_BARRIER_TIMEOUT_S="2", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", _ABSENT_PEER], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode != 0
    assert "NO TRAP" not in r.stdout
    assert "timed out waiting for rank 1" in r.stdout + r.stderr


def test_peer_exchange_with_every_token_on_one_rank():
    """Worst-case imbalance: every token picks experts 0 and 1, both on EP
    rank 0, so rank 0 receives all 4 ranks' rows (the receive buffers'
    worst-case capacity) and the other ranks' GEMMs get empty groups."""
    world, E, k, H, F, seed = 4, 8, 2, 128, 256, 21
    topo = B.ParallelTopology(world_size=world, ep=4)
    wg = -np.ones((H, E)) / H
    wg[:, 0] = 2.0 / H
    wg[:, 1] = 1.0 / H
    params = B.GatingParams(w_g=wg, k=k)
    weights = B.init_expert_weights(E, H, F, 1, seed, ep_size=4, activation="swiglu")
    rng = np.random.default_rng(seed)
    blocks, ups = [], []
    for r, n in enumerate((200, 160, 96, 256)):
        x = np.abs(rng.standard_normal((n, H))) + 0.1
        blocks.append(B.TokenBlock(torch.as_tensor(x, dtype=torch.float32).to("cuda", torch.bfloat16),
                                   np.arange(n) + 1000 * r))
        ups.append(torch.as_tensor(rng.standard_normal((n, H)), dtype=torch.float32).to("cuda", torch.bfloat16))
    o0, c0, r0 = _run("nccl", topo, params, weights, blocks, ups)
    o1, c1, r1 = _run("peer", topo, params, weights, blocks, ups)
    for r in range(world):
        assert set(c1.per_rank[r]["decision"].experts.unique().tolist()) == {0, 1}
        torch.testing.assert_close(o1[r], o0[r], rtol=0, atol=0)
        assert O.rel_err(r1.input_grads[r].float().cpu().numpy(),
                         r0.input_grads[r].float().cpu().numpy()) < 1e-2
    assert int(c1.per_rank[0]["pst"]["gcount"].sum()) == 2 * (200 + 160 + 96 + 256)
    assert int(c1.per_rank[1]["pst"]["gcount"].sum()) == 0
    for key in r0.expert_grads:
        for a, b in zip(r0.expert_grads[key][0] + r0.expert_grads[key][1],
                        r1.expert_grads[key][0] + r1.expert_grads[key][1]):
            assert O.rel_err(b.cpu().numpy(), a.cpu().numpy()) < 1e-3 or float(a.abs().max()) == 0.0


@pytest.mark.parametrize("world,ep,etp,E,k", [(2, 2, 1, 8, 4), (4, 4, 1, 16, 8), (4, 2, 2, 8, 2)])
def test_deduplicated_push_is_exact(world, ep, etp, E, k, monkeypatch):
    """One push per (token, remote EP index) with the duplicates resolved by
    the receiver (B200MOE_PUSH_DEDUP; default on from top-4 when an EP index
    hosts several experts) stores exactly the rows the per-pair push stores:
    outputs and every gradient are bit-identical with it on and off."""
    H, F, seed = 128, 256, 17
    topo = B.ParallelTopology(world_size=world, ep=ep, etp=etp, tp=etp)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k)
    weights = B.init_expert_weights(E, H, F, etp, seed, ep_size=ep, activation="swiglu")
    blocks, ups = _blocks((160, 96, 200, 64)[:world], H, seed)
    res = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("B200MOE_PUSH_DEDUP", flag)
        o, c, r = _run("peer", topo, params, weights, blocks, ups)
        assert c.per_rank[0]["peer"].dedup == (flag == "1")
        res[flag] = (o, r)
    (o1, r1), (o0, r0) = res["1"], res["0"]
    for r in range(world):
        torch.testing.assert_close(o1[r], o0[r], rtol=0, atol=0)
        torch.testing.assert_close(r1.input_grads[r], r0.input_grads[r], rtol=0, atol=0)
    torch.testing.assert_close(r1.w_g_grad, r0.w_g_grad, rtol=0, atol=0)
    for key in r0.expert_grads:
        for a, b in zip(r0.expert_grads[key][0] + r0.expert_grads[key][1],
                        r1.expert_grads[key][0] + r1.expert_grads[key][1]):
            torch.testing.assert_close(b, a, rtol=0, atol=0)


@pytest.mark.parametrize("nparts,k,E,H,dz,acc", [(1, 2, 8, 256, False, False), (2, 2, 8, 4096, False, False),
                                                 (2, 2, 8, 4096, True, False),
                                                 (3, 4, 8, 256, True, True), (2, 8, 64, 512, False, True),
                                                 (4, 1, 4, 136, True, False)])
def test_combine_parts_equals_reduce_then_combine(nparts, k, E, H, dz, acc):
    """ETP partial rows folded inside the combine (b200moe_combine_parts) give
    exactly ep_reduce_parts followed by the plain combine; the forward's
    materialised rows equal the reduced rows."""
    from paper_2504_14960_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(nparts * 100 + k)
    T, R = 300, 300 * k + 40
    parts = torch.randn((nparts, R, H), generator=g, device="cuda").to(torch.bfloat16)
    pair_row = torch.randperm(R, generator=g, device="cuda")[:T * k].to(torch.int32).reshape(T, k).contiguous()
    pair_row[5, 0] = -1  # a dropped pair
    gates = None if dz else torch.rand((T, k), generator=g, device="cuda")
    dzt = torch.randn((T, E), generator=g, device="cuda") if dz else None
    wgT = torch.randn((E, H), generator=g, device="cuda") * 0.05 if dz else None
    base = torch.randn((T, H), generator=g, device="cuda").to(torch.bfloat16)
    red = K.ep_reduce_parts(parts)
    want = K.combine(red, pair_row, T, gates=gates, dz=dzt, w_gT=wgT, out=base.clone() if acc else None,
                     accumulate=acc)
    rows_out = None if dz else torch.zeros((R, H), dtype=torch.bfloat16, device="cuda")
    got = K.combine(parts, pair_row, T, gates=gates, dz=dzt, w_gT=wgT, out=base.clone() if acc else None,
                    accumulate=acc, rows_out=rows_out)
    torch.testing.assert_close(got, want, rtol=0, atol=0)
    if rows_out is not None:
        used = pair_row[pair_row >= 0].long()
        torch.testing.assert_close(rows_out[used], red[used], rtol=0, atol=0)
