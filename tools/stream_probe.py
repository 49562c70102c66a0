"""Timeline probe of image_stream on cfg2: host wall per batch and the
device split (H2D stream vs compute stream) measured with CUDA events."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_00959_b200 as W  # noqa: E402

cfg = dict(bench.CFG2)
u, v, w, t, vis, wt = bench.synthetic(cfg)
spec = W.GridSpec(cfg["n_u"], cfg["n_v"], cfg["n_w"], cfg["cell"], w_max_native=cfg["w_max"])
kern = W.KernelSpec(cfg["kind"], cfg["S"], cfg["shape"])
pin = [torch.from_numpy(a).pin_memory() for a in (u, v, w, vis, wt)]
print("pinned:", [p.is_pinned() for p in pin], "from_numpy pinned:",
      torch.from_numpy(pin[0].numpy()).is_pinned())
batch = tuple(p.numpy() for p in pin)
dev = torch.device("cuda", 0)
# raw copy bandwidth of the 5 arrays on a side stream
s = torch.cuda.Stream(dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(s)
    d = [p.to(dev, non_blocking=True) for p in pin]
    e1.record(s)
torch.cuda.synchronize()
print("H2D side stream ms", e0.elapsed_time(e1))
for n in (1, 4, 8):
    t0 = time.perf_counter()
    k = 0
    for img, dg in W.image_stream([batch] * n, spec, kern):
        k += 1
    torch.cuda.synchronize()
    print(f"stream n={n}: {(time.perf_counter() - t0) * 1e3 / n:.2f} ms per batch")
t0 = time.perf_counter()
for _ in range(4):
    W.image(*batch[:3], None, *batch[3:], spec, kern)
print(f"single calls: {(time.perf_counter() - t0) * 1e3 / 4:.2f} ms per call")

# overlap experiment: H2D of one batch on a side stream while the device
# pipeline runs on resident inputs
dres = [p.to(dev) for p in pin]
W.image_device(*dres, spec, kern)
torch.cuda.synchronize()
stage = [torch.empty_like(x) for x in dres]
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for d_, p_ in zip(stage, pin):
            d_.copy_(p_, non_blocking=True)
    t1 = time.perf_counter()
    W.image_device(*dres, spec, kern)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"overlap rep {rep}: enqueue H2D {1e3*(t1-t0):.2f} ms, image_device {1e3*(t2-t1):.2f} ms, "
          f"total {1e3*(t3-t0):.2f} ms")
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for d_, p_ in zip(stage, pin):
            d_.copy_(p_, non_blocking=True)
    torch.cuda.synchronize()
    print(f"H2D alone {1e3*(time.perf_counter()-t0):.2f} ms")
print("current stream handle:", torch.cuda.current_stream().cuda_stream, "side:", s.cuda_stream)
