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
