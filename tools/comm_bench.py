"""NCCL all-to-all bandwidth on this box (torchrun, one rank per GPU).

Compares dist.all_to_all_single (one grouped send/recv per peer) against a
batch of per-(peer, expert) P2P chunks, at the MoE dispatch size (C2: 16384
tokens x top-2 x 4096 bf16 per rank).  Reports per-rank algorithmic bandwidth
(bytes leaving the rank / time) and nccl-tests busbw = algbw * (n-1)/n."""
import os
import time

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    rows, H = 32768, 4096
    send = torch.randn((rows, H), device=dev).to(torch.bfloat16)
    recv = torch.empty_like(send)
    split = [rows // world] * world
    chunks = 4

    def a2a():
        dist.all_to_all_single(recv, send, split, split)

    def p2p():
        ops = []
        per = rows // world // chunks
        for p in range(world):
            for c in range(chunks):
                off = p * (rows // world) + c * per
                if p == rank:
                    recv[off:off + per].copy_(send[off:off + per])
                    continue
                ops.append(dist.P2POp(dist.isend, send[off:off + per], p))
                ops.append(dist.P2POp(dist.irecv, recv[off:off + per], p))
        for r in dist.batch_isend_irecv(ops):
            r.wait()

    for name, fn in (("all_to_all_single", a2a), (f"p2p x{chunks}/peer", p2p)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
        off_bytes = send.numel() * send.element_size() * (world - 1) / world
        algbw = off_bytes / (ms / 1e3) / 1e9
        if rank == 0:
            print(f"{name}: world={world} {ms:.3f} ms  algbw(off-rank)={algbw:.1f} GB/s  "
                  f"busbw={send.numel() * 2 / (ms / 1e3) / 1e9 * (world - 1) / world:.1f} GB/s", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
