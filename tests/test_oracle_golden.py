"""Pin the CPU oracle (oracle/moe_oracle.py) to golden vectors produced by the
reference implementation itself (tests/golden/make_golden.py).

Integers (expert ids, kept masks, permutations, counts) must match exactly;
floats to 1e-12 relative (both sides are float64 numpy)."""
import numpy as np
import pytest

from oracle import moe_oracle as O


def _cases(d, prefix):
    return sorted({k.split("_")[0] for k in d if k.startswith(prefix)}, key=lambda s: int(s[1:]))


def test_router_cases_match_reference(golden):
    d = golden("router")
    cases = _cases(d, "r")
    assert len(cases) >= 10
    for c in cases:
        E, k, sig, renorm = (int(v) for v in d[c + "_meta"])
        r = O.route_logits(d[c + "_logits"], k, "sigmoid" if sig else "softmax", bool(renorm))
        np.testing.assert_array_equal(r.experts, d[c + "_experts"], err_msg=c)
        np.testing.assert_array_equal(r.gates, d[c + "_gates"], err_msg=c)
        np.testing.assert_array_equal(r.scores, d[c + "_scores"], err_msg=c)


def test_capacity_and_plan_cases_match_reference(golden):
    d = golden("capacity_plan")
    for c in _cases(d, "c"):
        E, k, n, prob = (int(v) for v in d[c + "_meta"])
        cf = float(d[c + "_cf"][0])
        r = O.route_logits(d[c + "_logits"], k)
        cap = O.capacity_limit(cf, n, E)
        assert cap == int(d[c + "_cap"][0])
        kept = O.apply_capacity(r.experts, r.gates, r.kept, np.arange(n), cap, E,
                                "probability" if prob else "position")
        np.testing.assert_array_equal(kept, d[c + "_kept"], err_msg=c)
        if not prob:
            np.testing.assert_array_equal(O.capacity_rank_vectorized(r.experts, cap, E), kept)
        for ep in (1, 2, 4):
            if c + f"_perm_ep{ep}" not in d:
                continue
            plan = O.build_dispatch_plan(r.experts, r.gates, kept, ep, E // ep)
            np.testing.assert_array_equal(plan.permutation, d[c + f"_perm_ep{ep}"])
            np.testing.assert_array_equal(plan.send_counts, d[c + f"_counts_ep{ep}"])
            np.testing.assert_array_equal(plan.gates, d[c + f"_pgates_ep{ep}"])
        plan = O.build_dispatch_plan(r.experts, r.gates, kept, 1, E)
        np.testing.assert_array_equal(O.permute(d[c + "_x"], plan), d[c + "_permuted"])
        np.testing.assert_allclose(O.unpermute_combine(d[c + "_rows"], plan, 8),
                                   d[c + "_combined"], rtol=0, atol=1e-13)


def test_expert_cases_match_reference(golden):
    d = golden("experts")
    for ci, act in enumerate(("relu", "gelu")):
        p = f"e{ci}_"
        ex = O.Expert(d[p + "w1"], d[p + "w2"], act)
        y, pre = O.expert_forward(d[p + "x"], ex)
        np.testing.assert_allclose(y, d[p + "y"], rtol=1e-12, atol=1e-13)
        dx, dw1, dw2 = O.expert_backward(d[p + "u"], d[p + "x"], pre, ex)
        for got, name in ((dx, "dx"), (dw1, "dw1"), (dw2, "dw2")):
            assert O.rel_err(got, d[p + name]) < 1e-12, name


def _layer_case(d, c):
    meta = [int(v) for v in d[c + "_meta"]]
    w, tp, cp, ep, etp, E, k, H, F, seq, batch, seed, full, sig, renorm, gelu = meta
    cf = float(d[c + "_cf"][0])
    cfg = O.LayerConfig(k=k, gate_fn="sigmoid" if sig else "softmax", renormalize=bool(renorm),
                        capacity_factor=None if cf < 0 else cf)
    experts = [O.Expert(d[c + "_w1"][e], d[c + "_w2"][e], "gelu" if gelu else "relu") for e in range(E)]
    return meta, cfg, experts


def test_layer_cases_match_reference(golden):
    """Per-rank oracle (full expert set, rank-local capacity scope) reproduces
    the reference's distributed moe_forward/moe_backward on every topology."""
    d = golden("layer")
    cases = _cases(d, "l")
    assert len(cases) >= 6
    for c in cases:
        meta, cfg, experts = _layer_case(d, c)
        w, E, k, seq, full = meta[0], meta[5], meta[6], meta[9], meta[12]
        x, u, wg = d[c + "_x"], d[c + "_u"], d[c + "_wg"]
        positions = [d[c + f"_positions{r}"] for r in range(w)]
        kept_over = [None] * w
        if full and cfg.capacity_factor is not None:
            routs = [O.route_logits(x[p] @ wg, k, cfg.gate_fn, cfg.renormalize) for p in positions]
            kept_over = O.full_sequence_kept([r.experts for r in routs], [r.gates for r in routs],
                                             positions, seq, cfg.capacity_factor, E)
        y = np.zeros_like(x)
        dx = np.zeros_like(x)
        dwg = np.zeros_like(wg)
        dw1 = [np.zeros_like(e.w1) for e in experts]
        dw2 = [np.zeros_like(e.w2) for e in experts]
        for r, pos in enumerate(positions):
            out, st = O.layer_forward(x[pos], x[pos] @ wg, experts, cfg, positions=pos,
                                      kept_override=kept_over[r])
            np.testing.assert_array_equal(st.routing.kept, d[c + "_kept"][pos], err_msg=c)
            np.testing.assert_array_equal(st.routing.experts, d[c + "_experts"][pos], err_msg=c)
            ep = meta[3]
            plan_ep = O.build_dispatch_plan(st.routing.experts, st.routing.gates, st.routing.kept,
                                            ep, E // ep)
            np.testing.assert_array_equal(plan_ep.permutation, d[c + f"_perm{r}"], err_msg=c)
            np.testing.assert_array_equal(plan_ep.send_counts, d[c + f"_counts{r}"], err_msg=c)
            y[pos] = out
            g = O.layer_backward(u[pos], st, experts, cfg, w_g=wg)
            dx[pos] = g[0]
            dwg += g[2]
            for e in range(E):
                dw1[e] += g[3][e]
                dw2[e] += g[4][e]
        assert O.rel_err(y, d[c + "_y"]) < 1e-12, c
        assert O.rel_err(dx, d[c + "_dx"]) < 1e-12, c
        assert O.rel_err(dwg, d[c + "_dwg"]) < 1e-12, c
        assert O.rel_err(np.stack(dw1), d[c + "_dw1"]) < 1e-12, c
        assert O.rel_err(np.stack(dw2), d[c + "_dw2"]) < 1e-12, c


# Known-answer tests the reference's own suite holds for this path, restated
# against the oracle (test_router.py / test_dispatcher.py / test_experts.py).

def test_known_answers():
    import math
    r = O.route_logits(np.array([[2.0, 0.0]]), 1)
    assert r.experts[0, 0] == 0 and abs(r.gates[0, 0] - math.exp(2) / (math.exp(2) + 1)) < 1e-15
    r = O.route_logits(np.zeros((4, 3)), 2)
    np.testing.assert_array_equal(r.experts, np.tile([0, 1], (4, 1)))
    r = O.route_logits(np.array([[0.5, -0.5]]), 1, "sigmoid")
    assert abs(r.gates[0, 0] - 1 / (1 + math.exp(-0.5))) < 1e-15
    assert O.capacity_limit(1.0, 8, 4) == 2 and O.capacity_limit(1.5, 8, 4) == 3
    assert O.capacity_limit(1.0, 2, 4) == 1
    ex = np.zeros((3, 1), dtype=np.int64)
    kept = O.apply_capacity(ex, np.ones((3, 1)), np.ones((3, 1), bool), np.arange(3), 2, 2)
    np.testing.assert_array_equal(kept.ravel(), [True, True, False])
    g = np.array([[0.1], [2.0], [1.0]])
    kept = O.apply_capacity(ex, g, np.ones((3, 1), bool), np.arange(3), 2, 2, "probability")
    np.testing.assert_array_equal(kept.ravel(), [False, True, True])
    plan = O.build_dispatch_plan(np.array([[0, 1]]), np.array([[0.6, 0.4]]), np.ones((1, 2), bool), 1, 2)
    u, v = np.array([[1.0, 0.0]]), np.array([[0.0, 1.0]])
    np.testing.assert_allclose(O.unpermute_combine(np.concatenate([u, v]), plan, 2), 0.6 * u + 0.4 * v)
    y, _ = O.expert_forward(np.array([[1.0]]), O.Expert(np.array([[2.0]]), np.array([[3.0]])))
    assert y[0, 0] == 6.0


@pytest.mark.parametrize("renorm", [False, True])
def test_swiglu_and_shared_backward_match_finite_differences(renorm):
    """Builder-defined SwiGLU + shared expert: analytic grads vs central FD
    (modelled on oracle.py:201-256), since the reference has no SwiGLU."""
    rng = np.random.default_rng(5)
    n, H, F, E, k = 12, 6, 5, 4, 2
    x = rng.standard_normal((n, H))
    wg = rng.standard_normal((H, E)) * 0.5
    u = rng.standard_normal((n, H))
    w1, w2 = O.swiglu_matrices(E, H, F, 3)
    experts = [O.Expert(a, b, "swiglu") for a, b in zip(w1, w2)]
    shared = O.Expert(*[m[0] for m in O.swiglu_matrices(1, H, 2 * F, 9)], act="swiglu")
    cfg = O.LayerConfig(k=k, renormalize=renorm)

    def loss(xv):
        y, _ = O.layer_forward(xv, xv @ wg, experts, cfg, shared=shared)
        return float((u * y).sum())

    _, st = O.layer_forward(x, x @ wg, experts, cfg, shared=shared)
    dx = O.layer_backward(u, st, experts, cfg, w_g=wg, shared=shared)[0]
    eps = 1e-6
    for idx in range(0, x.size, 7):
        xp = x.copy().ravel()
        xp[idx] += eps
        xm = x.copy().ravel()
        xm[idx] -= eps
        fd = (loss(xp.reshape(x.shape)) - loss(xm.reshape(x.shape))) / (2 * eps)
        assert abs(fd - dx.ravel()[idx]) < 1e-6 * max(1.0, abs(fd))
