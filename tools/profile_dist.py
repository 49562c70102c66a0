"""Phase timings of the multi-GPU path (run under torchrun): each stage of
image_distributed timed with a device synchronize + barrier around it."""

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
from paper_2504_00959_b200 import distributed as WD  # noqa: E402


class Timed(WD.CudaBackend):
    def __init__(self):
        super().__init__()
        self.t = {}

    def _wrap(self, name, fn, *a):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a)
        torch.cuda.synchronize()
        self.t[name] = self.t.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
        return out

    def prepare(self, *a):
        return self._wrap("prepare", super().prepare, *a)

    def route(self, *a):
        return self._wrap("route", super().route, *a)

    def grid_slab(self, *a):
        return self._wrap("grid_slab", super().grid_slab, *a)

    def fft_rows(self, *a):
        return self._wrap("fft_rows", super().fft_rows, *a)

    def fft_cols_stack(self, *a):
        return self._wrap("fft_cols", super().fft_cols_stack, *a)


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    cfg = dict(bench.CFG2)
    u, v, w, t, vis, wt = bench.synthetic(cfg, seed=cfg["seed"] + rank)
    dev = torch.device("cuda", local)
    arrs = [torch.from_numpy(a).to(dev) for a in (u, v, w, vis, wt)]
    spec = W.GridSpec(cfg["n_u"], cfg["n_v"], cfg["n_w"], cfg["cell"], w_max_native=cfg["w_max"])
    kern = W.KernelSpec("gaussian", 3, 1.0)
    be = Timed()
    for it in range(4):
        be.t = {}
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        WD.image_distributed(*arrs, spec, kern, backend=be, to_host=False)
        torch.cuda.synchronize()
        tot = (time.perf_counter() - t0) * 1e3
        if it == 3:
            print(f"rank {rank}: total {tot:.2f} ms, stages " +
                  ", ".join(f"{k} {v:.2f}" for k, v in be.t.items()) +
                  f", collectives+host {tot - sum(be.t.values()):.2f}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
