import os, sys, time, warnings, traceback
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2504_14960_b200 as B
from paper_2504_14960_b200 import dispatcher as D
cfgs = {"c4": (64, 8, 3584, 2560, 16384, 20480), "c2": (8, 2, 4096, 14336, 16384, 0)}
E, k, H, F, T, S_ = cfgs[sys.argv[1]]
dev = torch.device("cuda", 0)
topo = B.ParallelTopology(world_size=1)
rng = np.random.default_rng([0, 0]); bnd = 1.0 / np.sqrt(H)
wg = torch.as_tensor(rng.uniform(-bnd, bnd, size=(H, E)), dtype=torch.float32)
params = B.GatingParams(w_g=wg, k=k)
g = torch.Generator(device=dev).manual_seed(1)
w1 = [((torch.rand((H, 2 * F), generator=g, device=dev) * 2 - 1) * bnd) for _ in range(E)]
w2 = [((torch.rand((F, H), generator=g, device=dev) * 2 - 1) * bnd) for _ in range(E)]
weights = B.ExpertWeights(tuple(range(E)), w1, w2, "swiglu", 0, 1)
weights.packed(torch.bfloat16, dev)
shared = None
if S_:
    shared = B.ExpertWeights((0,), [(torch.rand((H, 2 * S_), generator=g, device=dev) * 2 - 1) * bnd],
                             [(torch.rand((S_, H), generator=g, device=dev) * 2 - 1) * bnd], "swiglu", 0, 1)
    shared.packed(torch.bfloat16, dev)
groups = B.generate_parallel_groups(topo)
nw = B.LocalWorld(1, dev); ctx = B.collectives.LocalRankContext(nw, 0)
layer = D.RankLayer(params, weights, topo, D._rank_groups(topo, groups, 0), 0, torch.bfloat16, dev, shared=shared)
x = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
u = torch.randn((T, H), generator=g, device=dev).to(torch.bfloat16)
pos = torch.arange(T)
def step():
    out, sv = layer.forward(ctx, x, pos)
    layer.backward(ctx, u, sv)
for _ in range(3): step()
torch.cuda.synchronize()
t0 = time.perf_counter(); step(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"host enqueue {1e3*(t1-t0):.2f} ms, total {1e3*(t2-t0):.2f} ms", flush=True)
torch.cuda.set_sync_debug_mode(1)
warnings.simplefilter("always")
def hook(message, category, filename, lineno, file=None, line=None):
    print("SYNC:", message, flush=True)
    traceback.print_stack(limit=12)
warnings.showwarning = hook
step()
torch.cuda.set_sync_debug_mode(0)
