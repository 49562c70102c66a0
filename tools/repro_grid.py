"""Debug helper: one dirty image at a given size (python tools/repro_grid.py N n_u n_w)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2504_00959_b200 as W

n, nu, nw = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(1)
u, v, w = rng.random(n), rng.random(n), rng.random(n)
vis = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
wt = np.ones(n, np.float32)
dev = torch.device("cuda", 0)
spec = W.GridSpec(nu, nu, nw, 0.4 / nu, w_max_native=100.0)
kern = W.KernelSpec.gaussian(3, 1.0)
args = [torch.from_numpy(a).to(dev) for a in (u, v, w, vis, wt)]
try:
    img, d = W.image_device(*args, spec, kern)
    torch.cuda.synchronize()
    print("ok", n, nu, nw, d["grid_updates"], d["tile_entries"], flush=True)
except Exception as e:
    print("FAIL", n, nu, nw, e, flush=True)
