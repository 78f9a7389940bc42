"""Tensor-core grouped GEMM (tcgen05/TMEM/TMA) against a float64 torch
reference on the same bf16 inputs, for every operand-major / grouping /
epilogue combination the expert FFN uses, including ragged and empty groups."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2504_14960_b200 import experts as X  # noqa: E402
from paper_2504_14960_b200 import gemm_tc, kernels as K  # noqa: E402

ALIGN = 128


@pytest.fixture(params=["1", "2"], ids=["cta1", "cta2"], autouse=True)
def cta_group(request, monkeypatch):
    """Run every test with single-CTA (128x256) and CTA-pair (256x256,
    tcgen05.mma.cta_group::2) tiles."""
    monkeypatch.setenv("B200MOE_CTA_GROUP", request.param)
    return request.param


def _layout(counts, align=ALIGN):
    pad = [(c + align - 1) // align * align for c in counts]
    off = np.concatenate(([0], np.cumsum(pad))).astype(np.int32)
    return off, pad


def _tokens(counts, width, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    off, _ = _layout(counts)
    x = torch.zeros((int(off[-1]), width), device="cuda", dtype=torch.bfloat16)
    for e, c in enumerate(counts):
        x[off[e]:off[e] + c] = torch.randn((c, width), generator=g, device="cuda").to(torch.bfloat16)
    return x, torch.as_tensor(off, device="cuda")


def _rel(got, want):
    return float((got.double() - want).abs().max() / want.abs().max().clamp_min(1e-30))


COUNTS = [300, 0, 129, 1000, 128, 7]


@pytest.mark.parametrize("N,K", [(256, 512), (384, 200), (1024, 1024), (136, 64)])
def test_grouped_m_kmajor_b(N, K):
    """C = X W^T per group (forward GEMMs: W stored [L, N, K])."""
    x, goff = _tokens(COUNTS, K, 1)
    L_ = len(COUNTS)
    w = (torch.randn((L_, N, K), device="cuda") / K ** 0.5).to(torch.bfloat16)
    c = torch.full((x.shape[0], N), 7.0, device="cuda", dtype=torch.bfloat16)
    gemm_tc.gemm(x, w, c, grouped_dim=0, G=L_, M=0, N=N, K=K, a_sm=K, a_sk=1, b_sg=N * K, b_sk=1,
                 b_sn=K, c_sg=0, ldc=N, group_off=goff, max_rows=x.shape[0])
    torch.cuda.synchronize()
    off = goff.cpu().numpy()
    for e in range(L_):
        if off[e + 1] == off[e]:
            continue
        want = x[off[e]:off[e + 1]].double() @ w[e].double().T
        assert _rel(c[off[e]:off[e + 1]], want) < 1e-2, (e, _rel(c[off[e]:off[e + 1]], want))


@pytest.mark.parametrize("N,K", [(256, 512), (512, 256), (320, 128)])
def test_grouped_m_mnmajor_b(N, K):
    """C = X W per group with W stored [L, K, N] (backward dgrad GEMMs)."""
    x, goff = _tokens(COUNTS, K, 2)
    L_ = len(COUNTS)
    w = (torch.randn((L_, K, N), device="cuda") / K ** 0.5).to(torch.bfloat16)
    c = torch.zeros((x.shape[0], N), device="cuda", dtype=torch.bfloat16)
    gemm_tc.gemm(x, w, c, grouped_dim=0, G=L_, M=0, N=N, K=K, a_sm=K, a_sk=1, b_sg=K * N, b_sk=N,
                 b_sn=1, c_sg=0, ldc=N, group_off=goff, max_rows=x.shape[0])
    torch.cuda.synchronize()
    off = goff.cpu().numpy()
    for e in range(L_):
        if off[e + 1] == off[e]:
            continue
        want = x[off[e]:off[e + 1]].double() @ w[e].double()
        assert _rel(c[off[e]:off[e + 1]], want) < 1e-2, e


@pytest.mark.parametrize("M,N", [(256, 256), (384, 512), (136, 264)])
def test_grouped_k_wgrad(M, N):
    """C_g = A_g^T B_g over each group's rows (weight gradients), fp32 out;
    an empty group must produce zeros."""
    a, goff = _tokens(COUNTS, M, 3)
    b, _ = _tokens(COUNTS, N, 4)
    G = len(COUNTS)
    c = torch.full((G, M, N), 3.0, device="cuda", dtype=torch.float32)
    gemm_tc.gemm(a, b, c, grouped_dim=1, G=G, M=M, N=N, K=0, a_sm=1, a_sk=M, b_sg=0, b_sk=N,
                 b_sn=1, c_sg=M * N, ldc=N, group_off=goff, max_rows=a.shape[0])
    torch.cuda.synchronize()
    off = goff.cpu().numpy()
    for g in range(G):
        want = a[off[g]:off[g + 1]].double().T @ b[off[g]:off[g + 1]].double()
        if off[g + 1] == off[g]:
            assert float(c[g].abs().max()) == 0.0
            continue
        assert _rel(c[g], want) < 1e-3, g


@pytest.mark.parametrize("act", ["swiglu", "relu", "gelu"])
def test_fused_ffn_epilogues_match_simt(act):
    """Tensor-core FFN (fused activation epilogues) == SIMT FFN on identical
    bf16 inputs, forward and backward."""
    H, F, E = 256, 192, 4
    counts = [200, 0, 77, 513]
    xp, goff = _tokens(counts, H, 5)
    dyp, _ = _tokens(counts, H, 6)
    rng = np.random.default_rng(0)
    n1 = 2 * F if act == "swiglu" else F
    w1 = [rng.uniform(-1, 1, (H, n1)) / H ** 0.5 for _ in range(E)]
    w2 = [rng.uniform(-1, 1, (F, H)) / H ** 0.5 for _ in range(E)]
    pk = X.pack_experts(w1, w2, act, torch.bfloat16, "cuda")
    R = xp.shape[0]
    outs = {}
    for mode in ("tc", "simt"):
        import os
        os.environ["B200MOE_DISABLE_TC"] = "1" if mode == "simt" else "0"
        try:
            pre, h, y = X.ffn_forward(xp, goff, E, None, pk, R)
            dxp, dw1, dw2 = X.ffn_backward(dyp, xp, pre, h, goff, E, None, pk, R)
        finally:
            os.environ["B200MOE_DISABLE_TC"] = "0"
        torch.cuda.synchronize()
        outs[mode] = (pre, h, y, dxp, dw1, dw2)
    for name, a_, b_ in zip(("pre", "h", "y", "dx", "dw1", "dw2"), outs["tc"], outs["simt"]):
        err = _rel(a_.float(), b_.double())
        assert err < 2e-2, (act, name, err)
