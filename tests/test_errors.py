"""The drop-in rejects what the reference rejects, with the same exception
classes.

Each test names the reference test it mirrors.  Host-side validation runs
before any device work, so those cases run without a GPU; the ones that need
device data (routing decisions, expert caches, non-finite checks) are marked
gpu."""
import numpy as np
import pytest
import torch

import paper_2504_14960_b200 as B
from paper_2504_14960_b200.errors import NumericError, ProtocolError, ValidationError


# ---------------------------------------------------------------- host side
def test_gating_params_validation():
    # test_router.py:116-122 (CF < 1), router.py:49-66 (k range, enums)
    w = np.ones((2, 4))
    with pytest.raises(ValidationError) as e:
        B.GatingParams(w_g=w, k=1, capacity_factor=0.5)
    assert e.value.constraint == "capacity_factor>=1"
    for k in (0, 5):
        with pytest.raises(ValidationError, match="k must satisfy"):
            B.GatingParams(w_g=w, k=k)
    with pytest.raises(ValidationError, match="gate_fn"):
        B.GatingParams(w_g=w, k=1, gate_fn="relu")
    with pytest.raises(ValidationError, match="drop_mode"):
        B.GatingParams(w_g=w, k=1, drop_mode="global")
    with pytest.raises(ValidationError, match="drop_priority"):
        B.GatingParams(w_g=w, k=1, drop_priority="random")
    with pytest.raises(ValidationError, match="2-D"):
        B.GatingParams(w_g=np.ones(4), k=1)


def test_expert_weight_divisibility():
    # test_experts.py:54-58
    with pytest.raises(ValidationError):
        B.init_expert_weights(2, 4, 6, etp_size=4, seed=0)
    with pytest.raises(ValidationError):
        B.init_expert_weights(3, 4, 8, etp_size=1, seed=0, ep_size=2)
    with pytest.raises(ValidationError, match="activation"):
        B.init_expert_weights(2, 4, 8, etp_size=1, seed=0, activation="tanh")


def test_token_partition_indivisible():
    # test_dispatcher.py:147-150
    with pytest.raises(ValidationError):
        B.token_partition(B.ParallelTopology(world_size=4, tp=4), seq_len=6, batch=1)


def test_layer_rejects_pp_and_bad_ep():
    # test_dispatcher.py:238-242 (pp), dispatcher.py:262-287 (ep | E, seq_len)
    params = B.GatingParams(w_g=np.ones((4, 2)), k=1)
    with pytest.raises(ValidationError, match="pp"):
        B.moe_forward([], {}, B.ParallelTopology(world_size=2, pp=2), params, B.LocalWorld(2, "cpu"))
    params3 = B.GatingParams(w_g=np.ones((4, 3)), k=1)
    with pytest.raises(ValidationError, match="divide"):
        B.moe_forward([None, None], {}, B.ParallelTopology(world_size=2, ep=2), params3,
                      B.LocalWorld(2, "cpu"))
    full = B.GatingParams(w_g=np.ones((4, 2)), k=1, capacity_factor=1.0, drop_mode="fullsequence")
    with pytest.raises(ValidationError, match="seq_len"):
        B.moe_forward([None], {}, B.ParallelTopology(world_size=1), full, B.LocalWorld(1, "cpu"))
    with pytest.raises(ValidationError, match="blocks"):
        B.moe_forward([None], {}, B.ParallelTopology(world_size=2), params, B.LocalWorld(2, "cpu"))


def test_var_buffer_validation():
    # test_collectives.py:306-313
    with pytest.raises(ValidationError):
        B.VarBuffer(torch.zeros(5), 2, [2])
    with pytest.raises(ValidationError):
        B.VarBuffer(torch.zeros(4), 2, [3, -1])


def test_collective_misuse_is_a_protocol_error():
    # test_collectives.py:73-89: mismatched count vectors name the rank
    world = B.LocalWorld(2, "cpu")

    def bad_counts(ctx):
        counts = [1, 1] if ctx.rank == 0 else [2]
        ctx.all_to_all_v((0, 1), B.VarBuffer.from_rows(torch.zeros((2, 1)), counts))

    with pytest.raises(ProtocolError, match="rank 1"):
        world.run(bad_counts)

    def outsider(ctx):
        ctx.all_to_all_v((0,), B.VarBuffer.from_rows(torch.zeros((1, 1)), [1]))

    with pytest.raises(ProtocolError, match="not part of"):
        B.LocalWorld(2, "cpu").run(outsider)


# ---------------------------------------------------------------- device side
@pytest.mark.gpu
def test_non_finite_tokens_rejected():
    # test_router.py:61-64
    p = B.GatingParams(w_g=np.ones((2, 2)), k=1)
    with pytest.raises(NumericError):
        B.compute_gates(np.array([[np.nan, 0.0]]), p)
    with pytest.raises(NumericError):
        B.compute_gates(np.array([[np.inf, 0.0]]), p)
    with pytest.raises(ValidationError, match="incompatible"):
        B.compute_gates(np.ones((3, 5)), p)


@pytest.mark.gpu
def test_expert_out_of_range_in_plan():
    # test_dispatcher.py:95-103
    dec = B.RoutingDecision(torch.tensor([[5]], device="cuda"), torch.ones((1, 1), device="cuda"),
                            torch.ones((1, 1), dtype=torch.bool, device="cuda"), torch.arange(1))
    with pytest.raises(ValidationError):
        B.build_dispatch_plan(dec, 2, 2)


@pytest.mark.gpu
def test_expert_shard_errors():
    # test_experts.py:86-90 (wrong expert id), :154-159 (upstream shape)
    w = B.ExpertWeights((0,), [np.ones((2, 32))], [np.ones((32, 2))], "relu", 0, 1)
    with pytest.raises(ValidationError):
        B.expert_forward_shard(np.ones((1, 2)), w, 3)
    _, cache = B.expert_forward_shard(np.ones((4, 2)), w, 0)
    with pytest.raises(ValidationError):
        B.expert_backward_shard(np.ones((3, 2)), cache, w, 0)


@pytest.mark.gpu
def test_layer_upstream_shape_mismatch():
    # test_dispatcher.py:318-325
    topo = B.ParallelTopology(world_size=2, ep=2)
    H, E = 64, 4
    params = B.GatingParams(w_g=B.init_gating_matrix(H, E, 0), k=2)
    weights = B.init_expert_weights(E, H, 128, 1, 0, ep_size=2)
    _, blocks = B.fabricate_token_blocks(topo, 64, 2, H, 0)
    _, ups = B.fabricate_upstream(topo, 64, 2, H, 0)
    outs, ctx = B.moe_forward(blocks, weights, topo, params, B.LocalWorld(2))
    with pytest.raises(ValidationError):
        B.moe_backward([u[:-1] for u in ups], ctx)
    with pytest.raises(ValidationError, match="upstream blocks"):
        B.moe_backward(ups[:1], ctx)
