"""One (or a few) device-resident steps of the cfg2 hot path, for ncu.

    python tools/profile_step.py [--steps 1] [--n 10000000] [--kind gaussian|kaiser_bessel] [--S 3]
"""

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_00959_b200 as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--nu", type=int, default=2048)
    ap.add_argument("--nw", type=int, default=32)
    ap.add_argument("--kind", default="gaussian")
    ap.add_argument("--S", type=int, default=3)
    ap.add_argument("--cell", type=float, default=None)
    ap.add_argument("--precision", type=int, default=64)
    a = ap.parse_args()
    cfg = dict(bench.CFG2, n_vis=a.n, n_u=a.nu, n_v=a.nu, n_w=a.nw)
    if a.cell:
        cfg["cell"] = a.cell
    u, v, w, t, vis, wt = bench.synthetic(cfg)
    dev = torch.device("cuda", 0)
    du, dv, dw, dvis, dwt = (torch.from_numpy(x).to(dev) for x in (u, v, w, vis, wt))
    spec = W.GridSpec(cfg["n_u"], cfg["n_v"], cfg["n_w"], cfg["cell"], w_max_native=cfg["w_max"])
    kern = (W.KernelSpec.gaussian(a.S, 1.0) if a.kind == "gaussian" else W.KernelSpec.kaiser_bessel(a.S))
    for _ in range(a.steps):
        img, diag = W.image_device(du, dv, dw, dvis, dwt, spec, kern, precision=a.precision)
    torch.cuda.synchronize()
    ms, n = W.last_timings(dev)
    print("kernel ms [prepare, bucket, grid, rows, cols, finish]:", [round(x, 3) for x in ms],
          "launches", n, "updates", diag["grid_updates"], "entries", diag["tile_entries"])


if __name__ == "__main__":
    main()
