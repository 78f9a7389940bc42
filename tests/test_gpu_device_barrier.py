"""GPU: the production synchronisation path of the peer exchange on ONE GPU.

LocalWorld(device_barrier=True) runs every rank on its own CUDA stream and
meets the ranks in ep_barrier_kernel (flag stores with st.release.sys into
the peers' buffers, ld.acquire.sys spin) instead of a host rendezvous: the
same kernels, flags and cross-rank stores the NcclWorld path uses across
GPUs -- the counts push into the peers' matrices, the dispatch push into
their receive buffers, the GEMM scatter epilogue writing into the senders'
return buffers and the deduplicated rows read by ep_expand after the
barrier.  Results must be bit-identical with the host-barrier emulation
(whose parity with the NCCL path and the oracle test_gpu_peer.py checks)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import moe_oracle as O  # noqa: E402

import paper_2504_14960_b200 as B  # noqa: E402
from paper_2504_14960_b200.errors import NumericError, ProtocolError, ValidationError  # noqa: E402


def _blocks(sizes, H, seed, nan_rank=None):
    rng = np.random.default_rng(seed)
    out, ups, start = [], [], 0
    for r, n in enumerate(sizes):
        x = rng.standard_normal((n, H))
        if r == nan_rank:
            x[n // 2, 1] = np.nan
        out.append(B.TokenBlock(torch.as_tensor(x, dtype=torch.float32).to("cuda", torch.bfloat16),
                                np.arange(start, start + n)))
        start += n
        ups.append(torch.as_tensor(rng.standard_normal((n, H)), dtype=torch.float32).to("cuda", torch.bfloat16))
    return out, ups


def _run(world, topo, params, weights, blocks, ups, shared=None):
    outs, ctx = B.moe_forward(blocks, weights, topo, params, world, dtype=torch.bfloat16,
                              shared_weights=shared)
    res = B.moe_backward(ups, ctx)
    ctx.check()
    torch.cuda.synchronize()
    return outs, ctx, res


def _same(a, b):
    (o0, c0, r0), (o1, c1, r1) = a, b
    for r in range(len(o0)):
        torch.testing.assert_close(o1[r], o0[r], rtol=0, atol=0)
        torch.testing.assert_close(r1.input_grads[r], r0.input_grads[r], rtol=0, atol=0)
    torch.testing.assert_close(r1.w_g_grad, r0.w_g_grad, rtol=0, atol=0)
    for key in r0.expert_grads:
        for x, y in zip(r0.expert_grads[key][0] + r0.expert_grads[key][1],
                        r1.expert_grads[key][0] + r1.expert_grads[key][1]):
            torch.testing.assert_close(y, x, rtol=0, atol=0)


CASES = [
    # world, ep, etp, E, k, sizes, cf, dedup
    (2, 2, 1, 8, 2, (384, 256), None, "0"),
    (2, 2, 1, 16, 4, (320, 192), None, "1"),  # deduplicated push across "ranks" (k >= 4, L >= 2)
    (4, 4, 1, 16, 8, (256, 96, 200, 160), None, "1"),  # k = 8, four experts per rank
    (4, 2, 2, 8, 2, (192, 64, 128, 256), 1.0, "0"),  # EP x ETP with dropping (C3-like)
    (4, 2, 2, 16, 4, (128, 128, 96, 64), None, "1"),  # dedup with ETP siblings
    (8, 8, 1, 8, 2, (96, 128, 64, 160, 32, 128, 96, 64), None, "0"),  # C2 at EP8: one expert per rank
    (2, 2, 1, 16, 4, (0, 256), None, "1"),  # a rank with an empty token block
]


@pytest.mark.parametrize("world,ep,etp,E,k,sizes,cf,dedup", CASES)
def test_device_barrier_matches_host_barrier(world, ep, etp, E, k, sizes, cf, dedup, monkeypatch):
    monkeypatch.setenv("B200MOE_PUSH_DEDUP", dedup)
    H, F, seed = 128, 256, 5
    topo = B.ParallelTopology(world_size=world, ep=ep, etp=etp, tp=etp)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k, capacity_factor=cf)
    weights = B.init_expert_weights(E, H, F, etp, seed, ep_size=ep, activation="swiglu")
    blocks, ups = _blocks(sizes, H, seed)
    host = _run(B.LocalWorld(world), topo, params, weights, blocks, ups)
    dw = B.LocalWorld(world, device_barrier=True)
    dev = _run(dw, topo, params, weights, blocks, ups)
    px = dev[1].per_rank[0]["peer"]
    assert px.device_barrier and px.epoch > 0 and px.dedup == (dedup == "1")
    _same(host, dev)
    # a second step on the same buffers (epochs advance, flags reused)
    _same(host, _run(dw, topo, params, weights, blocks, ups))


def test_dedup_on_off_bit_identical_with_device_barrier(monkeypatch):
    H, F, E, k, seed = 128, 256, 16, 4, 9
    topo = B.ParallelTopology(world_size=2, ep=2)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k)
    weights = B.init_expert_weights(E, H, F, 1, seed, ep_size=2, activation="swiglu")
    blocks, ups = _blocks((300, 200), H, seed)
    got = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("B200MOE_PUSH_DEDUP", flag)
        got[flag] = _run(B.LocalWorld(2, device_barrier=True), topo, params, weights, blocks, ups)
    _same(got["0"], got["1"])


def test_failed_step_fails_every_rank_then_recovers():
    """A non-finite block on one rank, then an oversized block: every rank
    finishes the step's device barriers (abort markers in the count rows),
    moe_forward raises the root cause, and the next step is unaffected."""
    H, F, E, k, seed = 128, 256, 8, 2, 3
    topo = B.ParallelTopology(world_size=2, ep=2)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k)
    weights = B.init_expert_weights(E, H, F, 1, seed, ep_size=2, activation="swiglu")
    blocks, ups = _blocks((128, 128), H, seed)
    ref = _run(B.LocalWorld(2), topo, params, weights, blocks, ups)
    for barrier in (False, True):
        world = B.LocalWorld(2, device_barrier=barrier)
        _run(world, topo, params, weights, blocks, ups)
        # raised by moe_forward when the step's status has landed, else by the
        # next synchronisation point (moe_backward of that step)
        bad, _ = _blocks((128, 128), H, seed, nan_rank=1)
        with pytest.raises(NumericError, match="rank 1"):
            _run(world, topo, params, weights, bad, ups)
        big, big_ups = _blocks((256, 128), H, seed)
        with pytest.raises(ValidationError, match="peer buffers"):
            _run(world, topo, params, weights, big, big_ups)
        _same(ref, _run(world, topo, params, weights, blocks, ups))
        # a flagged step whose backward never runs is raised by the next forward
        try:
            B.moe_forward(bad, weights, topo, params, world, dtype=torch.bfloat16)
            pending = True
        except NumericError:
            pending = False
        if pending:
            with pytest.raises(NumericError, match="rank 1"):
                B.moe_forward(blocks, weights, topo, params, world, dtype=torch.bfloat16)
        _same(ref, _run(world, topo, params, weights, blocks, ups))



def test_push_mode_must_agree(monkeypatch):
    """B200MOE_PUSH_DEDUP is agreed when the buffers are created; members that
    disagree fail loudly instead of leaving stale duplicate rows."""
    H, F, E, k, seed = 64, 128, 16, 4, 1
    topo = B.ParallelTopology(world_size=2, ep=2)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k)
    weights = B.init_expert_weights(E, H, F, 1, seed, ep_size=2, activation="swiglu")
    blocks, _ = _blocks((64, 64), H, seed)
    import threading

    orig = B.dispatcher.os.environ.get
    local = threading.local()

    def per_rank_env(key, default=None):
        if key == "B200MOE_PUSH_DEDUP":
            return "1" if getattr(local, "rank", 0) == 0 else "0"
        return orig(key, default)

    real = B.dispatcher.RankLayer._peer

    def tagged(self, ctx, T):
        local.rank = ctx.rank
        return real(self, ctx, T)

    monkeypatch.setattr(B.dispatcher.RankLayer, "_peer", tagged)
    monkeypatch.setattr(B.dispatcher.os.environ, "get", per_rank_env)
    with pytest.raises(ProtocolError, match="PUSH_DEDUP"):
        B.moe_forward(blocks, weights, topo, params, B.LocalWorld(2), dtype=torch.bfloat16)


def test_shared_expert_side_stream_is_exact(monkeypatch):
    """The shared expert's GEMMs on the side stream (overlapping the barrier
    waits after the routed GEMMs) give exactly the in-line results, with the
    device barrier and ranks on their own streams."""
    H, F, E, k, S, seed = 128, 256, 16, 4, 384, 4
    topo = B.ParallelTopology(world_size=2, ep=2)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k)
    weights = B.init_expert_weights(E, H, F, 1, seed, ep_size=2, activation="swiglu")
    shared = B.init_shared_expert(H, S, seed)
    blocks, ups = _blocks((256, 192), H, seed)
    got = {}
    for side in (False, True):
        monkeypatch.setattr(B.dispatcher, "_SIDE_SHARED", side)
        got[side] = _run(B.LocalWorld(2, device_barrier=True), topo, params, weights, blocks, ups,
                         shared=shared)
    _same(got[False], got[True])
    for a, b in zip(got[False][2].shared_grads, got[True][2].shared_grads):
        torch.testing.assert_close(a, b, rtol=0, atol=0)


def test_smaller_receive_buffers_and_clean_overflow():
    """peer_capacity sizes the receive buffers for f x the balanced load
    instead of the worst case; a step whose routing overflows them fails on
    every rank with ProtocolError (no trap) and the next step runs."""
    H, F, E, k, T, seed = 128, 256, 8, 2, 256, 6
    topo = B.ParallelTopology(world_size=2, ep=2)
    weights = B.init_expert_weights(E, H, F, 1, seed, ep_size=2, activation="swiglu")
    # feature 0 steers the routing: +1 -> experts 0, 1 (rank 0); -1 -> 4, 5 (rank 1)
    wg = np.zeros((H, E))
    wg[0, 0], wg[0, 1], wg[0, 4], wg[0, 5] = 2.0, 1.0, -2.0, -1.0
    params = B.GatingParams(w_g=wg, k=k)
    rng = np.random.default_rng(seed)

    def blocks_with(signs):
        out = []
        for r, sgn in enumerate(signs):
            x = rng.standard_normal((T, H)) * 0.1
            x[:, 0] = sgn
            out.append(B.TokenBlock(torch.as_tensor(x, dtype=torch.float32).to("cuda", torch.bfloat16),
                                    np.arange(r * T, (r + 1) * T)))
        return out

    ups = [torch.randn((T, H), device="cuda").to(torch.bfloat16) for _ in range(2)]
    split = blocks_with((1.0, -1.0))  # 512 rows to each rank
    skew = blocks_with((1.0, 1.0))  # 1024 rows to rank 0
    ref = _run(B.LocalWorld(2), topo, params, weights, split, ups)
    for barrier in (False, True):
        world = B.LocalWorld(2, device_barrier=barrier)
        outs, ctx = B.moe_forward(split, weights, topo, params, world, dtype=torch.bfloat16, peer_capacity=1.0)
        res = B.moe_backward(ups, ctx)
        torch.cuda.synchronize()
        from paper_2504_14960_b200.peer import capacity_rows

        cap = ctx.per_rank[0]["peer"].cap
        from paper_2504_14960_b200.kernels import GEMM_ALIGN

        assert cap == capacity_rows(2, T, k, E // 2, GEMM_ALIGN, 1.0) < capacity_rows(2, T, k, E // 2, GEMM_ALIGN)
        _same(ref, (outs, ctx, res))
        with pytest.raises(ProtocolError, match="overflows the peer receive buffers"):
            _, c2 = B.moe_forward(skew, weights, topo, params, world, dtype=torch.bfloat16)
            B.moe_backward(ups, c2)
            c2.check()
        _same(ref, _run(world, topo, params, weights, split, ups))


@pytest.mark.parametrize("world,ep,etp,E,k,sizes,cf,dedup", CASES)
@pytest.mark.parametrize("device_barrier", [False, True])
def test_overlapped_push_bit_identical(world, ep, etp, E, k, sizes, cf, dedup, device_barrier, monkeypatch):
    """The push split into its local stores and an NVLink part on the
    exchange stream beside GEMM1 over the rank's own rows (the default) gives
    exactly the results of the push completing before one GEMM1 launch."""
    monkeypatch.setenv("B200MOE_PUSH_DEDUP", dedup)
    H, F, seed = 128, 256, 11
    topo = B.ParallelTopology(world_size=world, ep=ep, etp=etp, tp=etp)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k, capacity_factor=cf)
    weights = B.init_expert_weights(E, H, F, etp, seed, ep_size=ep, activation="swiglu")
    blocks, ups = _blocks(sizes, H, seed)
    got = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("B200MOE_PUSH_OVERLAP", flag)
        w = B.LocalWorld(world, device_barrier=device_barrier)
        got[flag] = _run(w, topo, params, weights, blocks, ups)
        layer_px = got[flag][1].per_rank[0]["peer"]
        # more than 4 ranks sharing one GPU run the push serially (dispatcher._overlap_fits)
        assert ("split" in got[flag][1].per_rank[0]["pst"]) == (flag == "1" and world <= 4)
        assert layer_px.device_barrier == device_barrier
        if flag == "1":  # a second step on the same buffers and streams
            _same(got["0"], _run(w, topo, params, weights, blocks, ups))
    _same(got["0"], got["1"])


def test_overlapped_push_all_local_and_all_remote(monkeypatch):
    """Edge split groups: every token of rank 0 routed to its own experts
    (empty remote part of its push) and every token of rank 1 routed away
    (empty local part), through the router, with the device barrier."""
    H, F, E, k, seed = 128, 256, 8, 2, 4
    topo = B.ParallelTopology(world_size=2, ep=2)
    wg = np.zeros((H, E))
    wg[0, :4] = 4.0   # feature 0 large -> experts 0..3 (rank 0)
    wg[0, 4:] = -4.0  # feature 0 very negative -> experts 4..7 (rank 1)
    wg[1:, :] = O.gating_matrix(H - 1, E, seed) * 0.01
    params = B.GatingParams(w_g=wg, k=k)
    weights = B.init_expert_weights(E, H, F, 1, seed, ep_size=2, activation="swiglu")
    blocks, ups = _blocks((192, 160), H, seed)
    blocks[0].values[:, 0] = 30.0   # rank 0's tokens -> rank 0's experts
    blocks[1].values[:, 0] = 30.0   # rank 1's tokens -> rank 0's experts too
    got = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("B200MOE_PUSH_OVERLAP", flag)
        got[flag] = _run(B.LocalWorld(2, device_barrier=True), topo, params, weights, blocks, ups)
    dec0 = got["1"][1].per_rank[0]["decision"]
    assert bool((dec0.experts < 4).all())
    dec1 = got["1"][1].per_rank[1]["decision"]
    assert bool((dec1.experts < 4).all())
    _same(got["0"], got["1"])
