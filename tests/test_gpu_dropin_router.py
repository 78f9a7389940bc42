"""The reference's router and expert tests with only the import swapped.

Ported from /root/reference/pkg/tests/test_router.py:28-217 and
tests/test_experts.py:27-160: ``moefold`` becomes ``paper_2504_14960_b200``
and the calls are unchanged (numpy inputs, SimWorld, GatingParams,
compute_gates / apply_capacity / gather_full_sequence_decision / load_stats,
init_expert_weights / expert_forward_shard / expert_backward_shard).
Results are CUDA tensors, read through ``.cpu().numpy()``.  Integer results
(expert ids, kept masks, counts) stay exact; the B200 path computes in fp32
where the reference computes in fp64, so float equalities the reference
checks to 1e-12..1e-15 are checked to fp32 rounding (rel 1e-6 for single
values, 1e-5 for GEMM results), and the expert finite-difference check uses
an fp32-sized step.  Hypothesis-driven cases run over fixed seeds.  Not
ported: TestSelectionInvariance (exercises the reference's numpy helpers
softmax_rows / select_topk, which are not part of its exported API).
"""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2504_14960_b200 import SimWorld  # noqa: E402
from paper_2504_14960_b200.errors import NumericError, ValidationError  # noqa: E402
from paper_2504_14960_b200.experts import (ExpertWeights, expert_backward_shard,  # noqa: E402
                                           expert_forward_shard, full_expert_matrices, init_expert_weights)
from paper_2504_14960_b200.router import (PRIORITY_PROBABILITY, GatingParams, apply_capacity,  # noqa: E402
                                          capacity_limit, compute_gates, gather_full_sequence_decision,
                                          load_stats)

F32 = 1e-6


def npy(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def params_for(w_g, k, **kw):
    return GatingParams(w_g=np.asarray(w_g, dtype=float), k=k, **kw)


class TestComputeGates:
    def test_single_expert_gate_is_one(self):
        p = params_for(np.ones((3, 1)), k=1)
        dec = compute_gates(np.random.default_rng(0).standard_normal((5, 3)), p)
        assert (npy(dec.experts) == 0).all()
        np.testing.assert_array_equal(npy(dec.gates), np.ones((5, 1)))

    def test_closed_form_softmax_value(self):
        w_g = np.array([[2.0, 0.0], [0.0, 0.0]])
        p = params_for(w_g, k=1)
        dec = compute_gates(np.array([[1.0, 0.0]]), p)
        assert npy(dec.experts)[0, 0] == 0
        expected = math.exp(2.0) / (math.exp(2.0) + 1.0)
        assert abs(float(npy(dec.gates)[0, 0]) - expected) < F32

    def test_full_support_gates_sum_to_one(self):
        rng = np.random.default_rng(1)
        p = params_for(rng.standard_normal((4, 2)), k=2)
        dec = compute_gates(rng.standard_normal((7, 4)), p)
        np.testing.assert_allclose(npy(dec.gates).sum(axis=1), np.ones(7), atol=F32)

    def test_tie_breaks_to_lower_expert_id(self):
        p = params_for(np.zeros((2, 3)), k=2)
        dec = compute_gates(np.ones((4, 2)), p)
        np.testing.assert_array_equal(npy(dec.experts), np.tile([0, 1], (4, 1)))

    def test_renormalize_topk(self):
        rng = np.random.default_rng(2)
        p = params_for(rng.standard_normal((4, 6)), k=3, renormalize_topk=True)
        dec = compute_gates(rng.standard_normal((5, 4)), p)
        np.testing.assert_allclose(npy(dec.gates).sum(axis=1), np.ones(5), atol=F32)

    def test_nonfinite_input_rejected(self):
        p = params_for(np.ones((2, 2)), k=1)
        with pytest.raises(NumericError):
            compute_gates(np.array([[np.nan, 0.0]]), p)

    def test_sigmoid_gate(self):
        p = params_for(np.array([[1.0, -1.0]]), k=1, gate_fn="sigmoid")
        dec = compute_gates(np.array([[0.5]]), p)
        assert abs(float(npy(dec.gates)[0, 0]) - 1.0 / (1.0 + math.exp(-0.5))) < F32


class TestApplyCapacity:
    def test_capacity_formula(self):
        assert capacity_limit(1.0, 8, 4) == 2
        assert capacity_limit(1.5, 8, 4) == 3
        assert capacity_limit(1.0, 2, 4) == 1

    def test_dropless_noop(self):
        p = params_for(np.ones((2, 4)), k=1)
        dec = compute_gates(np.random.default_rng(0).standard_normal((6, 2)), p)
        out = apply_capacity(dec, 6, 4, p)
        assert npy(out.kept).all()

    def test_position_priority_drops_latest(self):
        p = params_for(np.array([[5.0, 0.0]]), k=1, capacity_factor=1.0)
        dec = compute_gates(np.ones((3, 1)), p)
        assert (npy(dec.experts) == 0).all()
        out = apply_capacity(dec, 4, 2, p)
        np.testing.assert_array_equal(npy(out.kept).ravel(), [True, True, False])

    def test_probability_priority_keeps_largest_gates(self):
        p = params_for(np.array([[1.0, 0.0]]), k=1, capacity_factor=1.0, drop_priority=PRIORITY_PROBABILITY)
        x = np.array([[0.1], [2.0], [1.0]])
        dec = compute_gates(x, p)
        assert (npy(dec.experts) == 0).all()
        out = apply_capacity(dec, 4, 2, p)
        np.testing.assert_array_equal(npy(out.kept).ravel(), [False, True, True])

    def test_cf_below_one_rejected(self):
        with pytest.raises(ValidationError):
            params_for(np.ones((2, 2)), k=1, capacity_factor=0.5)

    @pytest.mark.parametrize("seed", [0, 1, 7, 123, 2**31 - 1])
    def test_drop_monotone_in_cf(self, seed):
        rng = np.random.default_rng(seed)
        w = rng.standard_normal((3, 4))
        x = rng.standard_normal((12, 3))
        lo = params_for(w, k=2, capacity_factor=1.0)
        hi = params_for(w, k=2, capacity_factor=2.0)
        kept_lo = npy(apply_capacity(compute_gates(x, lo), 12, 4, lo).kept)
        kept_hi = npy(apply_capacity(compute_gates(x, hi), 12, 4, hi).kept)
        assert (~kept_lo | kept_hi).all()


class TestFullSequenceGather:
    @staticmethod
    def _run(n_ranks, seq_len, make_local, params, num_experts):
        world = SimWorld(n_ranks)

        def program(ctx):
            local = make_local(ctx.rank)
            return gather_full_sequence_decision(ctx, tuple(range(n_ranks)), local, seq_len, num_experts, params)

        return world.run(program)

    def test_group_of_one_matches_local_capacity(self):
        p = params_for(np.array([[5.0, 0.0]]), k=1, capacity_factor=1.0)
        dec = compute_gates(np.ones((4, 1)), p)
        res = self._run(1, 4, lambda r: dec, p, 2)
        global_dec, local_dec = res[0]
        expected = apply_capacity(dec, 4, 2, p)
        np.testing.assert_array_equal(npy(local_dec.kept), npy(expected.kept))
        np.testing.assert_array_equal(npy(global_dec.positions), npy(dec.positions))

    def test_two_shards_capacity_applies_globally(self):
        p = params_for(np.array([[5.0, 0.0]]), k=1, capacity_factor=1.0)

        def make_local(rank):
            return compute_gates(np.ones((4, 1)), p, positions=np.arange(4) + 4 * rank)

        res = self._run(2, 8, make_local, p, 2)
        for rank in range(2):
            global_dec, local_dec = res[rank]
            assert int(npy(global_dec.kept).sum()) == 4
            np.testing.assert_array_equal(npy(global_dec.kept).ravel(), [True] * 4 + [False] * 4)
            np.testing.assert_array_equal(npy(local_dec.kept).ravel(), [True] * 4 if rank == 0 else [False] * 4)

    def test_agreement_without_overflow(self):
        rng = np.random.default_rng(7)
        w = rng.standard_normal((3, 4))
        p = params_for(w, k=1, capacity_factor=2.0)
        blocks = [rng.standard_normal((4, 3)) for _ in range(2)]
        locals_ = [compute_gates(blocks[r], p, positions=np.arange(4) + 4 * r) for r in range(2)]
        sub = [apply_capacity(d, 4, 4, p) for d in locals_]
        res = self._run(2, 8, lambda r: locals_[r], p, 4)
        for r in range(2):
            if npy(sub[r].kept).all() and npy(res[r][1].kept).all():
                np.testing.assert_array_equal(npy(sub[r].kept), npy(res[r][1].kept))


class TestLoadStats:
    def test_uniform_routing(self):
        p = params_for(np.eye(4) * 10.0, k=1)
        x = np.eye(4)[np.arange(8) % 4]
        stats = load_stats(compute_gates(x, p), 4)
        np.testing.assert_array_equal(stats.counts, [2, 2, 2, 2])
        assert stats.imbalance == 1.0
        assert abs(stats.aux_loss - 1.0) < F32

    def test_collapsed_routing_imbalance_is_e(self):
        p = params_for(np.array([[5.0, 0.0, 0.0, 0.0]]), k=1)
        stats = load_stats(compute_gates(np.ones((8, 1)), p), 4)
        assert stats.imbalance == 4.0

    def test_dropped_pairs_not_counted(self):
        p = params_for(np.array([[5.0, 0.0]]), k=1, capacity_factor=1.0)
        dec = apply_capacity(compute_gates(np.ones((4, 1)), p), 4, 2, p)
        assert load_stats(dec, 2).counts[0] == 2


# ------------------------------------------------------------ test_experts.py
def single_expert(w1, w2, activation="relu", etp_rank=0, etp_size=1):
    return ExpertWeights(expert_ids=(0,), w1=[np.asarray(w1, dtype=float)], w2=[np.asarray(w2, dtype=float)],
                         activation=activation, etp_rank=etp_rank, etp_size=etp_size)


class TestExpertInit:
    def test_etp1_shard_is_full_matrix(self):
        full_w1, full_w2 = full_expert_matrices(2, 4, 8, seed=3)
        sharded = init_expert_weights(2, 4, 8, etp_size=1, seed=3)
        np.testing.assert_array_equal(npy(sharded[(0, 0)].w1[0]), npy(full_w1[0]))
        np.testing.assert_array_equal(npy(sharded[(0, 0)].w2[1]), npy(full_w2[1]))

    def test_etp2_shards_reconstruct(self):
        full_w1, full_w2 = full_expert_matrices(3, 4, 8, seed=9)
        sharded = init_expert_weights(3, 4, 8, etp_size=2, seed=9)
        for e in range(3):
            w1_cat = np.concatenate([npy(sharded[(0, r)].w1[e]) for r in range(2)], axis=1)
            w2_cat = np.concatenate([npy(sharded[(0, r)].w2[e]) for r in range(2)], axis=0)
            np.testing.assert_array_equal(w1_cat, npy(full_w1[e]))
            np.testing.assert_array_equal(w2_cat, npy(full_w2[e]))

    def test_same_seed_identical(self):
        a = init_expert_weights(2, 4, 8, etp_size=2, seed=5)
        b = init_expert_weights(2, 4, 8, etp_size=2, seed=5)
        for key in a:
            for i in range(len(a[key].w1)):
                np.testing.assert_array_equal(npy(a[key].w1[i]), npy(b[key].w1[i]))

    def test_divisibility_enforced(self):
        with pytest.raises(ValidationError):
            init_expert_weights(2, 4, 6, etp_size=4, seed=0)
        with pytest.raises(ValidationError):
            init_expert_weights(3, 4, 8, etp_size=1, seed=0, ep_size=2)

    def test_ep_placement_contiguous(self):
        sharded = init_expert_weights(4, 2, 4, etp_size=1, seed=0, ep_size=2)
        assert sharded[(0, 0)].expert_ids == (0, 1)
        assert sharded[(1, 0)].expert_ids == (2, 3)


class TestExpertForward:
    def test_zero_input_relu_zero_output(self):
        w = single_expert(np.ones((3, 5)), np.ones((5, 3)))
        out, _ = expert_forward_shard(np.zeros((4, 3)), w, 0)
        np.testing.assert_array_equal(npy(out), np.zeros((4, 3)))

    def test_hand_arithmetic_1x1(self):
        w = single_expert([[2.0]], [[3.0]])
        out, _ = expert_forward_shard(np.array([[1.0]]), w, 0)
        assert float(npy(out)[0, 0]) == 6.0

    def test_shard_partials_sum_to_full(self):
        rng = np.random.default_rng(12)
        x = rng.standard_normal((6, 4))
        full = init_expert_weights(2, 4, 8, etp_size=1, seed=12)
        halves = init_expert_weights(2, 4, 8, etp_size=2, seed=12)
        for e in range(2):
            want = npy(expert_forward_shard(x, full[(0, 0)], e)[0])
            parts = [npy(expert_forward_shard(x, halves[(0, r)], e)[0]) for r in range(2)]
            np.testing.assert_allclose(parts[0] + parts[1], want, atol=1e-5)

    def test_wrong_expert_id_rejected(self):
        w = single_expert([[1.0]], [[1.0]])
        with pytest.raises(ValidationError):
            expert_forward_shard(np.ones((1, 1)), w, 3)

    @pytest.mark.parametrize("alpha,seed", [(0.0, 0), (0.5, 1), (3.0, 2), (10.0, 3)])
    def test_relu_homogeneity(self, alpha, seed):
        rng = np.random.default_rng(seed)
        w = single_expert(rng.standard_normal((3, 4)), rng.standard_normal((4, 3)))
        x = rng.standard_normal((2, 3))
        base = npy(expert_forward_shard(x, w, 0)[0]).astype(np.float64)
        scaled = npy(expert_forward_shard(alpha * x, w, 0)[0]).astype(np.float64)
        np.testing.assert_allclose(scaled, alpha * base, atol=1e-5 * max(1.0, alpha))


class TestExpertBackward:
    def test_zero_upstream_zero_grads(self):
        rng = np.random.default_rng(0)
        w = single_expert(rng.standard_normal((3, 4)), rng.standard_normal((4, 3)))
        out, cache = expert_forward_shard(rng.standard_normal((5, 3)), w, 0)
        dx, dw1, dw2 = expert_backward_shard(np.zeros(tuple(out.shape)), cache, w, 0)
        assert not npy(dx).any() and not npy(dw1).any() and not npy(dw2).any()

    @pytest.mark.parametrize("activation", ["relu", "gelu"])
    def test_matches_finite_differences(self, activation):
        # the reference's step (1e-6) is below an fp32 forward's resolution; a
        # 1e-3 central difference keeps fp32 noise ~1e-4 and rarely crosses a
        # ReLU kink
        rng = np.random.default_rng(42)
        hidden, ffn, n = 4, 8, 5
        w1 = rng.standard_normal((hidden, ffn)) * 0.3
        w2 = rng.standard_normal((ffn, hidden)) * 0.3
        x = rng.standard_normal((n, hidden))
        upstream = rng.standard_normal((n, hidden))
        w = single_expert(w1, w2, activation=activation)
        out, cache = expert_forward_shard(x, w, 0)
        dx, dw1, dw2 = (npy(g).astype(np.float64) for g in expert_backward_shard(upstream, cache, w, 0))

        def loss(xv, w1v, w2v):
            o, _ = expert_forward_shard(xv, single_expert(w1v, w2v, activation=activation), 0)
            return float((upstream * npy(o).astype(np.float64)).sum())

        eps = 1e-3
        for arr, grad, tag in ((x, dx, "x"), (w1, dw1, "w1"), (w2, dw2, "w2")):
            flat = arr.ravel()
            for idx in rng.choice(flat.size, size=min(10, flat.size), replace=False):
                orig = flat[idx]
                flat[idx] = orig + eps
                up = loss(x, w1, w2)
                flat[idx] = orig - eps
                down = loss(x, w1, w2)
                flat[idx] = orig
                fd = (up - down) / (2 * eps)
                assert abs(fd - grad.ravel()[idx]) < 2e-3 * max(1.0, abs(fd)), tag

    def test_etp2_token_grad_partials_sum(self):
        rng = np.random.default_rng(8)
        x = rng.standard_normal((6, 4))
        upstream = rng.standard_normal((6, 4))
        full = init_expert_weights(1, 4, 8, etp_size=1, seed=21)
        halves = init_expert_weights(1, 4, 8, etp_size=2, seed=21)
        _, cache_full = expert_forward_shard(x, full[(0, 0)], 0)
        dx_full = npy(expert_backward_shard(upstream, cache_full, full[(0, 0)], 0)[0])
        parts = []
        for r in range(2):
            _, cache = expert_forward_shard(x, halves[(0, r)], 0)
            parts.append(npy(expert_backward_shard(upstream, cache, halves[(0, r)], 0)[0]))
        np.testing.assert_allclose(parts[0] + parts[1], dx_full, atol=1e-5)

    def test_shape_mismatch_rejected(self):
        w = single_expert(np.ones((2, 3)), np.ones((3, 2)))
        _, cache = expert_forward_shard(np.ones((4, 2)), w, 0)
        with pytest.raises(ValidationError):
            expert_backward_shard(np.ones((3, 2)), cache, w, 0)
