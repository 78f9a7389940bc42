"""Pinned host <-> device copy bandwidth on cuda:0 (the e2e leg's copies).

    python tools/pcie_probe.py

128 MiB copies: host->device, device->host, and both directions at once on
two streams.
"""
import torch, time
dev = torch.device("cuda", 0)
n = 128 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device=dev)
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): fn()
    e1.record(); torch.cuda.synchronize()
    print(name, f"{10 * n / e0.elapsed_time(e1) / 1e6:.1f} GB/s", flush=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory(); d2 = torch.empty_like(d)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print("both directions", f"{2 * 10 * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s total", flush=True)
