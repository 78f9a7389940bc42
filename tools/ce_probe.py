"""NVLink peer bandwidth by mechanism (torchrun, >= 2 GPUs).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/ce_probe.py

Each rank moves `--mib` MiB to (push) or from (pull) its peers' symmetric
buffers, split evenly over the peers, one stream per peer: with
cudaMemcpyAsync (copy engines) or with an SM elementwise kernel whose stores
(push) or loads (pull) hit peer memory.  Prints per-GPU per-direction GB/s
on rank 0.
"""
import argparse
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as sm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=224)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    nbytes = a.mib << 20
    peers = [p for p in range(world) if p != rank]
    chunk = nbytes // len(peers) // 4096 * 4096
    buf = sm.empty(chunk * world, dtype=torch.uint8, device=dev)
    h = sm.rendezvous(buf, dist.group.WORLD)
    src = torch.randint(0, 255, (chunk * world,), dtype=torch.uint8, device=dev)
    views = {p: h.get_buffer(p, (chunk * world,), torch.uint8) for p in peers}
    streams = {p: torch.cuda.Stream(dev) for p in peers}

    dst_local = torch.empty_like(src)

    def run(n_split, mode="ce_push"):
        main_s = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(main_s)
        for p in peers:
            s = streams[p]
            s.wait_event(ev)
            with torch.cuda.stream(s):
                sub = chunk // n_split
                for i in range(n_split):
                    remote = views[p][rank * chunk + i * sub: rank * chunk + (i + 1) * sub]
                    local = src[p * chunk + i * sub: p * chunk + (i + 1) * sub]
                    here = dst_local[p * chunk + i * sub: p * chunk + (i + 1) * sub]
                    if mode == "ce_push":
                        remote.copy_(local, non_blocking=True)
                    elif mode == "ce_pull":
                        here.copy_(remote, non_blocking=True)
                    elif mode == "sm_push":  # elementwise kernel storing into peer memory
                        torch.bitwise_or(local.view(torch.int64), 0, out=remote.view(torch.int64))
                    else:  # sm_pull: elementwise kernel loading from peer memory
                        torch.bitwise_or(remote.view(torch.int64), 0, out=here.view(torch.int64))
            main_s.wait_stream(s)

    for mode, n_split in (("ce_push", 1), ("ce_push", 4), ("ce_pull", 1), ("sm_push", 1), ("sm_pull", 1)):
        ms = []
        for _ in range(a.reps):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(n_split, mode)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        ms.sort()
        t = ms[len(ms) // 2]
        if rank == 0:
            gbs = chunk * len(peers) / t / 1e6
            print(f"{mode} x{n_split:<2d} {chunk * len(peers) / 2**20:7.1f} MiB  {t * 1e3:8.1f} us  "
                  f"{gbs:7.1f} GB/s ({gbs / 900:5.1%} of 900)", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
