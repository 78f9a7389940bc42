"""Pinned host <-> device copy bandwidth of N ranks at once (torchrun) --
the e2e leg's host copies at N GPUs.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/host_copy_probe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    n = 128 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    d2 = torch.empty_like(d)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name in ("h2d", "d2h", "both"):
        for rep in range(2):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(10):
                if name in ("h2d", "both"):
                    with torch.cuda.stream(s1):
                        d.copy_(h, non_blocking=True)
                if name in ("d2h", "both"):
                    with torch.cuda.stream(s2):
                        h2.copy_(d2, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        res[name] = (2 if name == "both" else 1) * 10 * n / dt / 1e9
    t = torch.tensor([res["h2d"], res["d2h"], res["both"]], device=dev)
    allt = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(allt, t)
    if rank == 0:
        print(f"world={world}", flush=True)
        for r, v in enumerate(allt):
            print(f"  rank {r}: h2d {v[0]:.1f}  d2h {v[1]:.1f}  both {v[2]:.1f} GB/s", flush=True)
        tot = torch.stack(allt).sum(0)
        print(f"  aggregate: h2d {tot[0]:.1f}  d2h {tot[1]:.1f}  both {tot[2]:.1f} GB/s", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
