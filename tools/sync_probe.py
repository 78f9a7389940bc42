"""Host synchronisations in the public API's steady state (1 GPU): runs
moe_forward / moe_backward under torch's sync-debug "warn" mode and prints
every synchronising call (expected: none -- the status check is an event
query).

    python tools/sync_probe.py
"""
import os, sys, warnings, traceback
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2504_14960_b200 as B
torch.cuda.set_device(0)
E, k, H, F, T = 8, 2, 1024, 2048, 4096
params = B.GatingParams(w_g=np.random.default_rng(0).uniform(-0.03, 0.03, size=(H, E)), k=k)
weights = B.init_expert_weights(E, H, F, 1, 0, activation="swiglu")
x = torch.randn((T, H), device="cuda").to(torch.bfloat16)
u = torch.randn((T, H), device="cuda").to(torch.bfloat16)
topo = B.ParallelTopology(world_size=1)
w = B.LocalWorld(1)
pos = np.arange(T)
for _ in range(3):
    o, c = B.moe_forward([B.TokenBlock(x, pos)], weights, topo, params, w)
    B.moe_backward([u], c)
torch.cuda.synchronize()
torch.cuda.set_sync_debug_mode("warn")
with warnings.catch_warnings(record=True) as ws:
    warnings.simplefilter("always")
    for _ in range(2):
        o, c = B.moe_forward([B.TokenBlock(x, pos)], weights, topo, params, w)
        B.moe_backward([u], c)
torch.cuda.set_sync_debug_mode("default")
print("warnings:", len(ws))
for wn in ws[:10]:
    print(wn.filename, wn.lineno, str(wn.message)[:120])
