"""Multi-GPU (NCCL) parity: launches tests/dist_layer_check.py under torchrun
on every visible GPU (>= 2), skipped on a single-GPU box."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
def test_nccl_layer_matches_emulated_ranks():
    n = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29517",
           os.path.join(ROOT, "tests", "dist_layer_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(out.stdout[-4000:])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-4000:]


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
@pytest.mark.parametrize("ep,etp", [(2, 1), (1, 2)])
def test_in_process_multi_gpu_world_matches_single_device(ep, etp):
    """LocalWorld(devices=[0, 1]): the ranks run as threads on two GPUs and
    the peer exchange stores into the other GPU's buffers over NVLink; the
    result must equal the same program with both ranks on one GPU."""
    import numpy as np

    import paper_2504_14960_b200 as B
    from oracle import moe_oracle as O

    E, k, H, F, seq, seed = 8, 2, 128, 256, 256, 7
    topo = B.ParallelTopology(world_size=2, ep=ep, etp=etp, tp=etp)
    params = B.GatingParams(w_g=O.gating_matrix(H, E, seed), k=k)
    weights = B.init_expert_weights(E, H, F, etp, seed, ep_size=ep, activation="swiglu")
    _, blocks = B.fabricate_token_blocks(topo, seq, topo.dp, H, seed, dtype=torch.bfloat16)
    _, ups = B.fabricate_upstream(topo, seq, topo.dp, H, seed, dtype=torch.bfloat16)
    runs = []
    for world in (B.LocalWorld(2), B.LocalWorld(2, devices=[0, 1])):
        outs, ctx = B.moe_forward(blocks, weights, topo, params, world, dtype=torch.bfloat16)
        res = B.moe_backward(ups, ctx)
        assert all(ctx.per_rank[r].get("peer") is not None for r in range(2))
        runs.append((outs, res))
    (o0, r0), (o1, r1) = runs
    assert o1[1].device.index == 1
    for r in range(2):
        torch.testing.assert_close(o1[r].cpu(), o0[r].cpu(), rtol=0, atol=0)
        torch.testing.assert_close(r1.input_grads[r].cpu(), r0.input_grads[r].cpu(), rtol=0, atol=0)
    assert O.rel_err(r1.w_g_grad.cpu().numpy(), r0.w_g_grad.cpu().numpy()) < 1e-6
