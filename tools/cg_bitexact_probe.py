"""Are tcgen05 GEMM results bit-identical between CTA-pair (M = 256) and
single-CTA (M = 128) tiles?  Runs the grouped FFN GEMMs of a small routed
layout with B200MOE_CTA_GROUP=2 and =1 and compares every output bitwise."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_14960_b200 as B  # noqa: E402
from paper_2504_14960_b200 import experts as X  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    E, H, F = 4, 1024, 2048
    g = torch.Generator(device=dev).manual_seed(0)
    w1 = [torch.randn((H, 2 * F), generator=g, device=dev) * 0.03 for _ in range(E)]
    w2 = [torch.randn((F, H), generator=g, device=dev) * 0.03 for _ in range(E)]
    pk = B.ExpertWeights(tuple(range(E)), w1, w2, "swiglu", 0, 1).packed(torch.bfloat16, dev)
    rows = [640, 384, 1152, 896]  # multiples of 128, some with half-empty pair tiles
    goff = torch.tensor([0] + list(torch.tensor(rows).cumsum(0)), dtype=torch.int32, device=dev)
    R = int(goff[-1])
    x = torch.randn((R, H), generator=g, device=dev).to(torch.bfloat16)
    dy = torch.randn((R, H), generator=g, device=dev).to(torch.bfloat16)
    out = {}
    for cg in ("2", "1"):
        os.environ["B200MOE_CTA_GROUP"] = cg
        pre, h, y = X.ffn_forward(x, goff, E, None, pk, R)
        dxp, dw1, dw2 = X.ffn_backward(dy, x, pre, h, goff, E, None, pk, R)
        torch.cuda.synchronize()
        out[cg] = dict(pre=pre, h=h, y=y, dx=dxp, dw1=dw1, dw2=dw2)
    for k in out["2"]:
        a, b = out["2"][k].float(), out["1"][k].float()
        same = torch.equal(a, b)
        print(f"{k:4s} bit-identical: {same}   max |diff| {float((a - b).abs().max()):.3e}", flush=True)


if __name__ == "__main__":
    main()
