"""All-to-all bandwidth on one box: NCCL all_to_all_single vs direct peer
writes through torch symmetric memory (each rank copies its block for rank d
straight into d's receive buffer over NVLink). Run under torchrun."""
import os
import time

import torch
import torch.distributed as dist


def main():
    ws = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    for mb in (256, 1024, 2048):
        n = mb * 2**20 // 8
        n -= n % ws
        send = torch.randn(n, dtype=torch.float64, device=dev)
        recv = torch.empty_like(send)
        for _ in range(3):
            dist.all_to_all_single(recv, send)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        it = 5
        for _ in range(it):
            dist.all_to_all_single(recv, send)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        moved = n * 8 * (ws - 1) / ws
        if rank == 0:
            print(f"nccl a2a {mb} MiB/rank: {ms:.3f} ms, {moved / ms / 1e6:.1f} GB/s out per rank", flush=True)
    # symmetric memory peer writes
    try:
        import torch.distributed._symmetric_memory as symm
        mb = 1024
        n = mb * 2**20 // 8
        n -= n % ws
        blk = n // ws
        buf = symm.empty(n, dtype=torch.float64, device=dev)
        hdl = symm.rendezvous(buf, dist.group.WORLD)
        send = torch.randn(n, dtype=torch.float64, device=dev)
        peers = [hdl.get_buffer(d, (n,), torch.float64) for d in range(ws)]
        streams = [torch.cuda.Stream(dev) for _ in range(ws)]

        def once():
            cur = torch.cuda.current_stream(dev)
            for d in range(ws):
                s = streams[d]
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    peers[d][rank * blk:(rank + 1) * blk].copy_(send[d * blk:(d + 1) * blk],
                                                                non_blocking=True)
            for s in streams:
                cur.wait_stream(s)
            hdl.barrier()

        for _ in range(3):
            once()
        torch.cuda.synchronize()
        dist.barrier()
        e0.record()
        for _ in range(it):
            once()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        moved = n * 8 * (ws - 1) / ws
        if rank == 0:
            print(f"symm peer copies {mb} MiB/rank: {ms:.3f} ms, {moved / ms / 1e6:.1f} GB/s out per rank",
                  flush=True)
    except Exception as exc:
        if rank == 0:
            print("symmetric memory unavailable:", type(exc).__name__, exc)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
