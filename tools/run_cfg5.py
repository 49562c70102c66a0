"""BASELINE config 5: Kaiser-Bessel support 3/7/11 (half_support 1/3/5,
beta = 2.34 S) x FP32/FP64 on the 4096x4096x64 mesh, LOFAR-like tracks
(100M records by default), one GPU. Prints one JSON line per case: step
time, Mvis/s, kernel split, NVML energy per image and the FP32-vs-FP64
image difference (relative L2) -- the green-productivity comparison.

    python tools/run_cfg5.py [--records 100000000] [--steps 3]"""

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tools")]

import torch  # noqa: E402

import paper_2504_00959_b200 as W  # noqa: E402
from lofar import tracks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--records", type=int, default=100_000_000)
    ap.add_argument("--mesh", type=int, default=4096)
    ap.add_argument("--planes", type=int, default=64)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cell = 1e-4
    spec = W.GridSpec(a.mesh, a.mesh, a.planes, cell, w_max_native=1000.0)
    u, v, w, t, vis, wt = tracks(a.records, cell, device=dev)
    try:
        from paper_2504_00959_b200.energy import NvmlRaplMeter
        meter = NvmlRaplMeter(devices=[0], host=False)
    except Exception:
        meter = None
    img = torch.empty((a.mesh, a.mesh), dtype=torch.float64, device=dev)
    for S in (1, 3, 5):
        kern = W.KernelSpec.kaiser_bessel(S)
        ref = None
        for prec in (64, 32):
            W.image_device(u, v, w, vis, wt, spec, kern, image_out=img, precision=prec)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if meter:
                meter.start()
            e0.record()
            for _ in range(a.steps):
                _, d = W.image_device(u, v, w, vis, wt, spec, kern, image_out=img, precision=prec)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            joules = meter.joules()["gpu"] / a.steps if meter else None
            kms, _ = W.last_timings(dev)
            out = {"config": "cfg5", "kernel": f"kaiser_bessel S={S} (support {2 * S + 1})",
                   "beta": kern.shape_param, "precision": prec, "records": a.records,
                   "grid": [a.mesh, a.mesh, a.planes], "ms_per_step": round(ms, 3),
                   "mvis_s": round(a.records / ms / 1e3, 1),
                   "kernel_ms": [round(x, 3) for x in kms],
                   "gpu_joules_per_image": round(joules, 3) if joules else None,
                   "grid_updates": d["grid_updates"]}
            if prec == 64:
                ref = img.clone()
            else:
                out["rel_l2_vs_fp64"] = float(torch.linalg.norm(img - ref) / torch.linalg.norm(ref))
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
