"""GPU parity at BASELINE.json's full sizes (C2-C5, one rank per config).

The numpy oracle is too slow at these sizes (minutes per layer), so:
- routing, capacity and the dispatch plan are integer work: checked bit for
  bit against the oracle's functions on the GPU's own fp32 logits (cheap in
  numpy even at 16384 x 64);
- the floating-point layer (forward output, token / router / expert
  gradients) is checked against a plain PyTorch fp32 restatement of the same
  layer (oracle/moe_oracle.py's structure: layer_forward/layer_backward) run
  on the same bf16 inputs, bf16-rounded weights and routing, within the
  north star's bf16 tolerance (rel-err 2e-2);
- size-independent properties hold exactly: the backward is linear in the
  upstream gradient (scaling by 2 is exact in every dtype, so 2u gives
  exactly twice every gradient), runs are deterministic, outputs do not
  depend on how the tokens are split over EP ranks, and pad-to-capacity
  equals the unpadded layer.
"""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import moe_oracle as O  # noqa: E402

import paper_2504_14960_b200 as B  # noqa: E402
from paper_2504_14960_b200 import dispatcher as D  # noqa: E402

BF16_TOL = 2e-2

# BASELINE.json configs at per-rank size (SURVEY.md §8 notation)
CFGS = {
    "c2": dict(E=8, k=2, H=4096, F=14336, T=16384, S=0, cf=None),
    "c3": dict(E=8, k=2, H=4096, F=14336, T=16384, S=0, cf=1.0),
    "c4": dict(E=64, k=8, H=3584, F=2560, T=16384, S=20480, cf=None),
    "c5": dict(E=8, k=2, H=6144, F=16384, T=8192, S=0, cf=None),
}


class Layer:
    """One rank holding every expert of a config, inputs resident on cuda:0."""

    def __init__(self, name, seed=0, pad=False):
        c = CFGS[name]
        self.c = c
        E, H, F, T, S = c["E"], c["H"], c["F"], c["T"], c["S"]
        dev = torch.device("cuda", 0)
        g = torch.Generator(device=dev).manual_seed(seed)
        bnd = 1.0 / math.sqrt(H)

        def uni(*shape):
            return ((torch.rand(shape, generator=g, device=dev) * 2 - 1) * bnd).to(torch.bfloat16)

        # bf16 weights (the layer computes on bf16 operands; the fp32
        # reference below uses exactly these values)
        self.w1 = [uni(H, 2 * F) for _ in range(E)]  # [gate | up]
        self.w2 = [uni(F, H) for _ in range(E)]
        self.wg = O.gating_matrix(H, E, seed)
        self.params = B.GatingParams(w_g=self.wg, k=c["k"], capacity_factor=c["cf"])
        self.weights = B.ExpertWeights(tuple(range(E)), self.w1, self.w2, "swiglu", 0, 1)
        self.shared = None
        if S:
            self.sw1, self.sw2 = uni(H, 2 * S), uni(S, H)
            self.shared = B.ExpertWeights((0,), [self.sw1], [self.sw2], "swiglu", 0, 1)
        topo = B.ParallelTopology(world_size=1)
        groups = B.generate_parallel_groups(topo)
        self.layer = D.RankLayer(self.params, self.weights, topo, D._rank_groups(topo, groups, 0), 0,
                                 torch.bfloat16, dev, shared=self.shared, pad_to_capacity=pad)
        self.ctx = B.collectives.LocalRankContext(B.LocalWorld(1, dev), 0)
        self.x = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
        self.u = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
        self.pos = torch.arange(T, dtype=torch.int64)

    def run(self, u=None):
        out, sv = self.layer.forward(self.ctx, self.x, self.pos)
        dx, dwg, dw1p, dw2p = self.layer.backward(self.ctx, self.u if u is None else u, sv)
        torch.cuda.synchronize()
        return out, sv, (dx, dwg, dw1p, dw2p)


def _silu(z):
    return z * torch.sigmoid(z)


def _ffn_fp32(xe, w1, w2, dy=None):
    """SwiGLU FFN in fp32 (oracle.expert_forward/expert_backward structure):
    returns y, and with ``dy`` also (dx, dW1 [H, 2F], dW2 [F, H])."""
    F = w2.shape[0]
    w1f, w2f = w1.float(), w2.float()
    pre = xe @ w1f
    a, b = pre[:, :F], pre[:, F:]
    h = _silu(a) * b
    y = h @ w2f
    if dy is None:
        return y, None
    dw2 = h.T @ dy
    dh = dy @ w2f.T
    sa = torch.sigmoid(a)
    da = dh * b * (sa * (1 + a * (1 - sa)))
    db = dh * _silu(a)
    dpre = torch.cat([da, db], 1)
    return y, (dpre @ w1f.T, xe.T @ dpre, dw2)


def reference_layer(L: Layer, dec, u):
    """fp32 restatement of the layer (oracle.layer_forward / layer_backward,
    softmax gates, no renormalisation) on the GPU's routing decision."""
    x, uf = L.x.float(), u.float()
    T, H = x.shape
    experts, gates, kept = dec.experts.long(), dec.gates.float(), dec.kept.bool()
    scores = dec.scores.float()
    out = torch.zeros((T, H), device=x.device)
    dx = torch.zeros((T, H), device=x.device)
    dgates = torch.zeros_like(gates)
    dw1, dw2 = [], []
    for e in range(L.c["E"]):
        t_idx, s_idx = ((experts == e) & kept).nonzero(as_tuple=True)
        ge = gates[t_idx, s_idx][:, None]
        xe = x[t_idx]
        y, _ = _ffn_fp32(xe, L.w1[e], L.w2[e])
        y = y.to(torch.bfloat16).float()  # the layer returns bf16 expert rows
        out.index_add_(0, t_idx, ge * y)
        dgates[t_idx, s_idx] = (uf[t_idx] * y).sum(1)
        _, (dxe, g1, g2) = _ffn_fp32(xe, L.w1[e], L.w2[e], ge * uf[t_idx])
        dx.index_add_(0, t_idx, dxe)
        dw1.append(g1)
        dw2.append(g2)
    if L.shared is not None:
        ys, (dxs, _, _) = _ffn_fp32(x, L.sw1, L.sw2, uf)
        out += ys
        dx += dxs
    # softmax router backward (dispatcher.py:474-490)
    ds = torch.zeros_like(scores).scatter_(1, experts, dgates * kept)
    dz = scores * (ds - (ds * scores).sum(1, keepdim=True))
    wg = torch.as_tensor(L.wg, dtype=torch.float32, device=x.device)
    dx += dz @ wg.T
    return out, dx, x.T @ dz, dw1, dw2


def _rel(a, b):
    """max|a - b| / max|b| -- the north star's rel-err
    (reference tests/test_acceptance.py:85-87)."""
    a, b = a.double(), b.double()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def _record(name, errs):
    """Per-tensor errors, also appended to $B200MOE_PARITY_LOG (JSON lines)
    when set, for profiles/."""
    import json
    import os

    print(name, {k: f"{v:.2e}" for k, v in errs.items()})
    path = os.environ.get("B200MOE_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"config": name, "metric": "max|d|/max|want|", **errs}) + "\n")


def _layer_errors(L, out, sv, grads):
    dx, dwg, dw1p, dw2p = grads
    ro, rdx, rdwg, rdw1, rdw2 = reference_layer(L, sv["dec"], L.u)
    E = L.c["E"]
    return {"out": _rel(out.float(), ro), "dx": _rel(dx.float(), rdx), "dw_g": _rel(dwg.float(), rdwg),
            "dw1": max(_rel(dw1p[e].T.float(), rdw1[e]) for e in range(E)),
            "dw2": max(_rel(dw2p[e].T.float(), rdw2[e]) for e in range(E))}


@pytest.mark.parametrize("name", ["c2", "c4", "c5"])
def test_full_size_layer_vs_fp32_reference(name):
    L = Layer(name)
    out, sv, (dx, dwg, dw1p, dw2p) = L.run()
    dec = sv["dec"]
    # routing ints bit-exact against the oracle on the layer's own logits
    r = O.route_logits(sv["logits"].double().cpu().numpy(), L.c["k"])
    np.testing.assert_array_equal(dec.experts.cpu().numpy(), r.experts)
    assert O.rel_err(dec.gates.cpu().numpy(), r.gates) < 1e-6
    plan = O.build_dispatch_plan(r.experts, r.gates, r.kept, 1, L.c["E"])
    P = plan.permutation.size
    assert int(sv["plan_dev"].offsets[-1]) == P
    np.testing.assert_array_equal(sv["plan_dev"].perm[:P].cpu().numpy(), plan.permutation)
    np.testing.assert_array_equal(sv["plan_dev"].counts.cpu().numpy(), plan.send_counts.reshape(-1))
    # floats against the fp32 restatement
    errs = _layer_errors(L, out, sv, (dx, dwg, dw1p, dw2p))
    _record(name, errs)
    for key, v in errs.items():
        assert v < BF16_TOL, (key, v)


def test_full_size_backward_is_linear_and_deterministic():
    L = Layer("c2")
    out1, _, g1 = L.run()
    out2, _, g2 = L.run()
    _, _, g3 = L.run(u=L.u * 2)
    torch.testing.assert_close(out1, out2, rtol=0, atol=0)
    for a, b, c in zip(g1, g2, g3):
        torch.testing.assert_close(a, b, rtol=0, atol=0)  # run to run
        torch.testing.assert_close(c, a * 2, rtol=0, atol=0)  # linear in u, exactly


def test_full_size_outputs_independent_of_ep_split():
    """C2's tokens split over EP2 (exchange over the peer buffers, ranks as
    threads) give the same output rows, bit for bit, as one rank holding all
    experts (dispatcher.py:194-217's factorisation independence)."""
    L = Layer("c2")
    out1, _, _ = L.run()
    topo = B.ParallelTopology(world_size=2, ep=2)
    E = L.c["E"]
    wmap = {(0, 0): B.ExpertWeights(tuple(range(E // 2)), L.w1[:E // 2], L.w2[:E // 2], "swiglu", 0, 1),
            (1, 0): B.ExpertWeights(tuple(range(E // 2, E)), L.w1[E // 2:], L.w2[E // 2:], "swiglu", 0, 1)}
    T = L.c["T"]
    h = T // 2
    blocks = [B.TokenBlock(L.x[:h].contiguous(), torch.arange(h)),
              B.TokenBlock(L.x[h:].contiguous(), torch.arange(h, T))]
    outs, _ = B.moe_forward(blocks, wmap, topo, L.params, B.LocalWorld(2), dtype=torch.bfloat16,
                            exchange="peer", check_finite_inputs=False)
    torch.testing.assert_close(torch.cat(outs), out1, rtol=0, atol=0)


def test_full_size_capacity_and_padding():
    """C3 (CF 1.0, sub-sequence dropping): the kept mask equals the oracle's
    apply_capacity on the layer's own routing, every expert keeps at most
    cap = T/E pairs, and the pad-to-capacity layout gives the same output
    bit for bit."""
    L = Layer("c3")
    out, sv, grads = L.run()
    dec = sv["dec"]
    T, E, k = L.c["T"], L.c["E"], L.c["k"]
    cap = O.capacity_limit(1.0, T, E)
    experts = dec.experts.cpu().numpy().astype(np.int64)
    want = O.capacity_rank_vectorized(experts, cap, E)
    np.testing.assert_array_equal(dec.kept.cpu().numpy(), want)
    assert np.bincount(experts[want], minlength=E).max() <= cap
    # floats against the fp32 restatement on the kept pairs (dropped pairs
    # contribute nothing; fully dropped tokens output exact zeros)
    errs = _layer_errors(L, out, sv, grads)
    _record("c3", errs)
    for key, v in errs.items():
        assert v < BF16_TOL, (key, v)
    dropped = ~dec.kept.any(1)
    if bool(dropped.any()):
        assert not bool(out[dropped].any())
    P = Layer("c3", pad=True)
    out_p, sv_p, grads_p = P.run()
    torch.testing.assert_close(out_p, out, rtol=0, atol=0)
    errs_p = _layer_errors(P, out_p, sv_p, grads_p)
    _record("c3-pad-to-capacity", errs_p)
    for key, v in errs_p.items():
        assert v < BF16_TOL, (key, v)
    # gradients: same sums over the same rows (padding rows are zero)
    for a, b in zip(grads_p, grads):
        assert _rel(a.float(), b.float()) < 1e-6
