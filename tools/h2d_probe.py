"""Concurrent pinned host->device bandwidth, one process per GPU (torchrun):
is the multi-GPU e2e bound by the box's shared host link?"""
import os
import time

import torch
import torch.distributed as dist

dist.init_process_group("nccl")
r, ws = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
torch.cuda.set_device(dev)
h = torch.empty(360_000_000, dtype=torch.uint8).pin_memory()
d = torch.empty_like(h, device=dev)
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
dist.barrier()
t0 = time.perf_counter()
for _ in range(10):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
if r == 0:
    print(f"{ws} ranks: per-rank {10 * 0.36 / t.item():.1f} GB/s, aggregate {ws * 10 * 0.36 / t.item():.1f} GB/s")
dist.destroy_process_group()
