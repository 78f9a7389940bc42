"""GPU: the fp32 router GEMMs on the bf16 tensor cores (three exact bf16 parts
of W_g / dz) against float64 references and the CUDA-core kernels."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2504_14960_b200 import kernels as K  # noqa: E402
from paper_2504_14960_b200.router import GatingParams  # noqa: E402


def _rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return float((a - b).norm() / b.norm().clamp_min(1e-300))


@pytest.mark.parametrize("T,H,E", [(1000, 256, 8), (4096, 1024, 64), (333, 512, 4), (2048, 3584, 64)])
def test_split_parts_are_exact(T, H, E):
    g = torch.Generator(device="cuda").manual_seed(T + E)
    w = torch.randn((T, E), generator=g, device="cuda") * 3.0
    p3, p6 = K.split_bf16x3(w, want3=True, want6=True)
    Ep = (E + 7) // 8 * 8
    hi, mid, lo = (p3[:, i * Ep:i * Ep + E].double() for i in range(3))
    assert torch.equal((hi + mid + lo), w.double())
    order = (0, 0, 0, 1, 1, 2)
    for j, i in enumerate(order):
        assert torch.equal(p6[:, j * Ep:j * Ep + E], p3[:, i * Ep:i * Ep + E])


@pytest.mark.parametrize("T,H,E", [(1000, 256, 8), (4096, 1024, 64), (333, 512, 4), (2048, 3584, 64)])
def test_tensor_core_router_gemms_match_fp64(T, H, E):
    g = torch.Generator(device="cuda").manual_seed(7 * T + E)
    bnd = H ** -0.5
    wg = ((torch.rand((H, E), generator=g, device="cuda") * 2 - 1) * bnd).float()
    params = GatingParams(w_g=wg.cpu().numpy().astype(np.float64), k=min(2, E))
    parts = params.device_w_g_parts("cuda")
    x = torch.randn((T, H), generator=g, device="cuda").to(torch.bfloat16)
    dz = torch.randn((T, E), generator=g, device="cuda") * 10.0
    ref_logits = x.double() @ wg.double()
    got = K.router_logits(x, wg, parts=parts)
    assert _rel(got, ref_logits) < 1e-5  # tensor-core fp32 accumulation over K = H
    # the CUDA-core kernel, for scale: both are fp32-accurate
    assert _rel(K.router_logits(x, wg), ref_logits) < 2e-6
    # dx += dz W_g^T into a bf16 buffer
    base = torch.randn((T, H), generator=g, device="cuda").to(torch.bfloat16)
    out = base.clone()
    K.router_term(dz, wg, out, parts=parts)
    ref = base.double() + dz.double() @ wg.double().T
    assert _rel(out, ref) < 4e-3
    # dW_g = x^T dz (split-K over token chunks)
    dwg = K.router_wgrad(x, dz, tc=True)
    ref_w = x.double().T @ dz.double()
    assert _rel(dwg, ref_w) < 1e-5
    assert _rel(K.router_wgrad(x, dz), ref_w) < 2e-6


# ----------------------------------------------------------- fused router
from oracle import moe_oracle as O  # noqa: E402
from paper_2504_14960_b200 import _lib as L  # noqa: E402


@pytest.mark.parametrize("T,H,E,k", [(16384, 4096, 8, 2), (1000, 256, 8, 2), (333, 512, 4, 1),
                                     (2048, 3584, 64, 8), (777, 1024, 16, 4), (640, 512, 32, 6)])
@pytest.mark.parametrize("gate_fn,renorm", [("softmax", False), ("sigmoid", True)])
def test_fused_router_forward(T, H, E, k, gate_fn, renorm):
    """router_fwd (tcgen05 logits + softmax/sigmoid + top-k in one kernel,
    router_tc.cu): logits fp32-accurate against float64, and ids / scores /
    gates exactly the reference arithmetic on those logits (router.py:146-162),
    checked against the pinned oracle; ties injected."""
    g = torch.Generator(device="cuda").manual_seed(T * 31 + E)
    bnd = H ** -0.5
    wg = ((torch.rand((H, E), generator=g, device="cuda") * 2 - 1) * bnd).float()
    x = torch.randn((T, H), generator=g, device="cuda").to(torch.bfloat16)
    x[5::97] = x[5]  # identical rows: identical logits
    if E >= 2:
        wg[:, 1] = wg[:, 0]  # experts 0 and 1 tie on every token
    params = GatingParams(w_g=wg, k=k, gate_fn=gate_fn, renormalize_topk=renorm)
    st = torch.zeros((1,), dtype=torch.int32, device="cuda")
    code = L.GATE_SOFTMAX if gate_fn == "softmax" else L.GATE_SIGMOID
    logits, scores, idx, gates, g64 = K.router_fwd(x, params.device_w_g_tc("cuda"), E, k, code, renorm, st,
                                                   want_f64=True)
    torch.cuda.synchronize()
    assert int(st) == 0
    ref = x.double() @ wg.double()
    assert float((logits.double() - ref).abs().max() / ref.abs().max()) < 1e-5
    lg = logits.double().cpu().numpy()
    ro = O.route_logits(lg, k, gate_fn, renorm)
    np.testing.assert_array_equal(idx.cpu().numpy(), ro.experts)
    np.testing.assert_allclose(g64.cpu().numpy(), ro.gates, rtol=1e-14, atol=0)
    np.testing.assert_allclose(gates.cpu().numpy(), ro.gates.astype(np.float32), rtol=1e-6)
    np.testing.assert_allclose(scores.cpu().numpy(), ro.scores.astype(np.float32), rtol=1e-6, atol=1e-30)


def test_fused_router_flags_nonfinite_and_routes_safely():
    T, H, E, k = 1000, 512, 8, 2
    g = torch.Generator(device="cuda").manual_seed(3)
    wg = torch.randn((H, E), generator=g, device="cuda") * H ** -0.5
    x = torch.randn((T, H), generator=g, device="cuda").to(torch.bfloat16)
    x[17, 3] = float("nan")
    x[900, 0] = float("inf")
    params = GatingParams(w_g=wg, k=k)
    st = torch.zeros((1,), dtype=torch.int32, device="cuda")
    _, _, idx, _, _ = K.router_fwd(x, params.device_w_g_tc("cuda"), E, k, L.GATE_SOFTMAX, False, st)
    assert int(st) & 1
    assert idx[17].tolist() == [0, 1] and idx[900].tolist() == [0, 1]
    assert int(idx.min()) >= 0 and int(idx.max()) < E


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_layer_nonfinite_raises_without_blocking_check(dtype):
    """moe_forward raises NumericError (router.py:141-144) from the device flag;
    the message names the token block or the gating weights like the reference."""
    import paper_2504_14960_b200 as B
    from paper_2504_14960_b200.errors import NumericError

    E, k, H, F, T = 8, 2, 256, 512, 512
    params = B.GatingParams(w_g=O.gating_matrix(H, E, 0), k=k)
    weights = B.init_expert_weights(E, H, F, 1, 0, activation="swiglu")
    x = torch.randn((T, H), device="cuda").to(dtype)
    x[7, 5] = float("nan")
    u = [torch.randn((T, H), device="cuda").to(dtype)]
    topo = B.ParallelTopology(world_size=1)
    # raised by moe_forward if the step's status copy has landed, else by moe_backward
    with pytest.raises(NumericError, match="token block"):
        _, ctx = B.moe_forward([B.TokenBlock(x, np.arange(T))], weights, topo, params, B.LocalWorld(1))
        B.moe_backward(u, ctx)
        ctx.check()
    wbad = O.gating_matrix(H, E, 0)
    wbad[3, 2] = np.inf
    with pytest.raises(NumericError, match="gating weights"):
        _, ctx = B.moe_forward([B.TokenBlock(torch.randn((T, H), device="cuda").to(dtype), np.arange(T))],
                               weights, topo, B.GatingParams(w_g=wbad, k=k), B.LocalWorld(1))
        B.moe_backward(u, ctx)
        ctx.check()
    # a flagged forward without its backward is raised by the next forward on that world
    w1 = B.LocalWorld(1)
    try:
        B.moe_forward([B.TokenBlock(x, np.arange(T))], weights, topo, params, w1)
        pending = True
    except NumericError:
        pending = False
    if pending:
        with pytest.raises(NumericError):
            B.moe_forward([B.TokenBlock(x.nan_to_num(), np.arange(T))], weights, topo, params, w1)
    # unchecked: no error, valid routing
    outs, _ = B.moe_forward([B.TokenBlock(x, np.arange(T))], weights, B.ParallelTopology(world_size=1), params,
                            B.LocalWorld(1), check_finite_inputs=False)
    torch.cuda.synchronize()


@pytest.mark.parametrize("T,H,E,k,acc", [(16384, 4096, 8, 2, False), (1000, 6144, 8, 2, True),
                                         (333, 512, 4, 1, False), (777, 1032, 8, 4, True)])
def test_combine_with_router_term(T, H, E, k, acc):
    """Backward combine with the fused router term (dispatcher.py:480-490):
    dx = sum of the k pair rows + dz W_g^T (+ the shared-expert dx), bf16 out,
    against float64 on the same inputs; dropped pairs (-1) contribute nothing."""
    g = torch.Generator(device="cuda").manual_seed(T + H)
    R = T * k
    rows = torch.randn((R, H), generator=g, device="cuda").to(torch.bfloat16)
    pair_row = torch.randperm(R, generator=g, device="cuda").to(torch.int32).reshape(T, k).contiguous()
    pair_row[::7, -1] = -1
    dz = torch.randn((T, E), generator=g, device="cuda")
    wg = torch.randn((H, E), generator=g, device="cuda") * H ** -0.5
    base = torch.randn((T, H), generator=g, device="cuda").to(torch.bfloat16)
    out = base.clone() if acc else None
    dx = K.combine(rows, pair_row, T, dz=dz, w_gT=wg.T.contiguous(), out=out, accumulate=acc)
    pr = pair_row.long()
    ref = torch.zeros((T, H), dtype=torch.float64, device="cuda")
    for s in range(k):
        m = pr[:, s] >= 0
        ref[m] += rows[pr[m, s]].double()
    ref += dz.double() @ wg.double().T
    if acc:
        ref += base.double()
    err = float((dx.double() - ref).abs().max() / ref.abs().max())
    assert err < 8e-3, err  # one bf16 rounding of the result


@pytest.mark.parametrize("T,H,E,k", [(16384, 4096, 8, 2), (1000, 256, 8, 2), (333, 512, 4, 1),
                                     (2048, 3584, 64, 8), (777, 1024, 16, 4), (640, 512, 32, 6)])
def test_tensor_core_wgrad_from_dz_parts(T, H, E, k):
    """router_bwd writes dz and its exact bf16 parts; router_wgrad_tc
    (x^T dz on the tensor cores, x read once) matches float64 and the parts
    sum back to dz exactly."""
    g = torch.Generator(device="cuda").manual_seed(T * 3 + E)
    x = torch.randn((T, H), generator=g, device="cuda").to(torch.bfloat16)
    logits = torch.randn((T, E), generator=g, device="cuda")
    scores, idx, gates, _ = K.router_topk(logits, k, L.GATE_SOFTMAX, False)
    dgates = torch.randn((T, k), generator=g, device="cuda")
    dz, parts = K.router_bwd(dgates, scores, idx, gates, L.GATE_SOFTMAX, False, want_parts=True)
    torch.testing.assert_close(dz, K.router_bwd(dgates, scores, idx, gates, L.GATE_SOFTMAX, False),
                               rtol=0, atol=0)
    epw = next(c for c in (8, 16, 32, 64) if c >= E)
    p = parts.double()
    recon = p[:, :E] + p[:, epw:epw + E] + p[:, 2 * epw:2 * epw + E]
    assert torch.equal(recon, dz.double())
    pad = torch.ones(parts.shape[1], dtype=torch.bool, device="cuda")
    for q in range(3):
        pad[q * epw:q * epw + E] = False
    assert not bool(parts[:, pad].any())
    dwg = K.router_wgrad_tc(x, parts, E)
    ref = x.double().T @ dz.double()
    assert float((dwg.double() - ref).abs().max() / ref.abs().max()) < 1e-5
    # deterministic: the split reduction runs in a fixed order
    torch.testing.assert_close(K.router_wgrad_tc(x, parts, E), dwg, rtol=0, atol=0)
