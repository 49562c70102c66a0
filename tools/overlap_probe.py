"""Probe: how much do two independent cfg2 images overlap on one GPU when
their pipelines run on two contexts / streams (K1 and the FFT passes of one
image beside K2 of the other)? Prints ms per image sequential vs concurrent."""
import ctypes as C
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_00959_b200 as W  # noqa: E402
from paper_2504_00959_b200 import _lib as L  # noqa: E402

cfg = dict(bench.CFG2)
u, v, w, t, vis, wt = bench.synthetic(cfg)
spec = W.GridSpec(cfg["n_u"], cfg["n_v"], cfg["n_w"], cfg["cell"], w_max_native=cfg["w_max"])
kern = W.KernelSpec(cfg["kind"], cfg["S"], cfg["shape"])
dev = torch.device("cuda", 0)
d = [torch.from_numpy(a).to(dev) for a in (u, v, w)]
dvis = torch.from_numpy(vis.reshape(-1).view(np.float32).copy()).to(dev)
dwt = torch.from_numpy(wt.reshape(-1).copy()).to(dev)
n = d[0].numel()
g, k = spec.c_struct(), kern.c_struct()
lib = L.lib()


def run(ctx, img):
    L.check(lib.wsb_image_device(ctx.handle, C.byref(g), C.byref(k), *(C.c_void_p(x.data_ptr()) for x in d),
                                 C.c_void_p(dvis.data_ptr()), C.c_void_p(dwt.data_ptr()), n, 1,
                                 C.c_void_p(img.data_ptr()), None))


for prio in (0, -1):
    sa = torch.cuda.Stream(dev)
    sb = torch.cuda.Stream(dev, priority=prio)
    ca, cb = L.Context(0), L.Context(0)
    ca.bind_stream(sa.cuda_stream)
    cb.bind_stream(sb.cuda_stream)
    ia = torch.empty((spec.n_v, spec.n_u), dtype=torch.float64, device=dev)
    ib = torch.empty_like(ia)
    for _ in range(3):
        run(ca, ia)
        run(cb, ib)
    torch.cuda.synchronize()
    N = 10
    t0 = time.perf_counter()
    for _ in range(N):
        run(ca, ia)
    torch.cuda.synchronize()
    seq = (time.perf_counter() - t0) / N
    t0 = time.perf_counter()
    for _ in range(N):
        run(ca, ia)
        run(cb, ib)
    torch.cuda.synchronize()
    conc = (time.perf_counter() - t0) / (2 * N)
    print(f"priority {prio}: sequential {seq * 1e3:.3f} ms/image, two streams {conc * 1e3:.3f} ms/image")
