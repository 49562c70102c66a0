"""Wall time per distributed image (torchrun): device-resident records with
to_host False / True, against the device-timed step -- where the multi-GPU
e2e loses time beyond the per-rank H2D."""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2504_00959_b200 as W  # noqa: E402
import paper_2504_00959_b200.distributed as WD  # noqa: E402

dist.init_process_group("nccl")
r = dist.get_rank()
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
torch.cuda.set_device(dev)
cfg = dict(bench.CFG2)
u, v, w, t, vis, wt = bench.synthetic(cfg, seed=r)
spec = W.GridSpec(cfg["n_u"], cfg["n_v"], cfg["n_w"], cfg["cell"], w_max_native=cfg["w_max"])
kern = W.KernelSpec(cfg["kind"], cfg["S"], cfg["shape"])
d = [torch.from_numpy(a).to(dev) for a in (u, v, w, vis, wt)]
for to_host in (False, True):
    for _ in range(3):
        WD.image_distributed(*d, spec, kern, to_host=to_host)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(10):
        WD.image_distributed(*d, spec, kern, to_host=to_host)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 10 * 1e3
    x = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    if r == 0:
        print(f"to_host={to_host}: {x.item():.2f} ms wall per image", flush=True)
dist.destroy_process_group()
