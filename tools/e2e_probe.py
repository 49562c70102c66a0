"""Phase split of the host-buffer entry (wsb_image) on the cfg2 workload:
H2D, device pipeline, D2H and wall time per call."""
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
pin = [torch.from_numpy(a).pin_memory().numpy() for a in (u, v, w, vis, wt)]
for it in range(4):
    t0 = time.perf_counter()
    img, d = W.image(pin[0], pin[1], pin[2], None, pin[3], pin[4], spec, kern)
    wall = (time.perf_counter() - t0) * 1e3
    print(f"wall {wall:.2f} ms  phase_ms {[round(x, 3) for x in d['phase_ms']]}", flush=True)
