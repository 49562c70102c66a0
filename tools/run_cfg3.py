"""BASELINE config 3 (north star): 100M LOFAR-like track records,
4096x4096x64, Gaussian support 7, FP64. Single process (1 GPU) or torchrun
(v-slab over N GPUs). cfg4 (SKA-scale) is the same driver with
--records 1000000000 --mesh 16384 --planes 32 --cell 1e-5 on 4-8 GPUs. Prints kernel/step timings and a linearity check
(image(a + b) == image(a) + image(b) within FP64 roundoff), a property that
holds at any size."""

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tools")]

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2504_00959_b200 as W  # noqa: E402
from lofar import tracks  # noqa: E402


STAGES = ("prepare", "route", "exchange", "grid", "bucket", "sweep", "rows", "cols", "gather",
          "fft", "reduce")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--records", dest="n", type=int, default=100_000_000)
    ap.add_argument("--mesh", dest="nu", type=int, default=4096)
    ap.add_argument("--planes", dest="nw", type=int, default=64)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--cell", type=float, default=1e-4)
    ap.add_argument("--transpose", default="auto", choices=["auto", "push", "peer", "nccl"])
    ap.add_argument("--decomp", default="auto", choices=["auto", "slabs", "planes"])
    ap.add_argument("--plane-weight-div", type=float, default=None,
                    help="plane decomposition: plane weight = n_u n_v / this (default: library's)")
    ap.add_argument("--label", default="cfg3 LOFAR-like tracks")
    a = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
        from paper_2504_00959_b200.distributed import image_distributed
    cell = a.cell
    pw = None if a.plane_weight_div is None else a.nu * a.nu / a.plane_weight_div
    spec = W.GridSpec(a.nu, a.nu, a.nw, cell, w_max_native=1000.0)
    kern = W.KernelSpec.gaussian(3, 1.0)
    per = a.n // ws
    t0 = time.perf_counter()
    u, v, w, t, vis, wt = tracks(a.n, cell, first=rank * per, count=per, device=dev)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0

    def run(vv=vis):
        if ws > 1:
            img, d = image_distributed(u, v, w, vv, wt, spec, kern, to_host=False, transpose=a.transpose,
                                           decomposition=a.decomp, plane_weight=pw)
            return (img.pixels if img is not None else None), d
        return W.image_device(u, v, w, vv, wt, spec, kern)

    run()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        pix, d = run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    if ws > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    out = {"config": a.label, "records": a.n, "grid": [a.nu, a.nu, a.nw],
           "n_gpus": ws, "ms_per_step": round(ms, 3), "mvis_s": round(a.n / ms / 1e3, 1),
           "grid_updates": d["grid_updates"], "generate_s": round(gen_s, 2)}
    if ws == 1:
        kms, _ = W.last_timings(dev)
        out["kernel_ms"] = [round(x, 3) for x in kms]
    else:
        tm = {}
        image_distributed(u, v, w, vis, wt, spec, kern, to_host=False, timings=tm,
                          transpose=a.transpose, decomposition=a.decomp, plane_weight=pw)
        st = torch.tensor([tm.get(k, 0.0) for k in STAGES], device=dev, dtype=torch.float64)
        per = [torch.empty_like(st) for _ in range(ws)]
        dist.all_gather(per, st)
        out["stage_ms_per_rank"] = {k: [round(float(p_[i]), 2) for p_ in per]
                                    for i, k in enumerate(STAGES) if k in tm}
        dist.all_reduce(st, op=dist.ReduceOp.MAX)
        out["stage_ms_max_over_ranks"] = {k: round(float(x), 3) for k, x in zip(STAGES, st.tolist())
                                          if k in tm}
        out["decomposition"] = a.decomp
        if "plane_starts" in d:
            out["plane_starts"] = d["plane_starts"]
    if a.check:
        # Size-independent parity at full size (linearity of the whole path):
        # split the records into two complementary halves by zeroing the
        # other half's weights; image(all) = image(A) + image(B) to FP64
        # rounding, and both halves plus the whole keep the exact update
        # count relation (the taps do not depend on the weights).
        g = torch.Generator(device=dev).manual_seed(7)
        mask = torch.rand(wt.shape, generator=g, device=dev) < 0.5
        wa = torch.where(mask, wt, torch.zeros_like(wt))
        wb = torch.where(mask, torch.zeros_like(wt), wt)

        def run_w(wts):
            if ws > 1:
                img, d = image_distributed(u, v, w, vis, wts, spec, kern, to_host=False,
                                           decomposition=a.decomp, plane_weight=pw)
                return (img.pixels.clone() if img is not None else None), d
            pix, d = W.image_device(u, v, w, vis, wts, spec, kern)
            return pix.clone(), d

        pall, dall = run_w(wt)
        pa, _ = run_w(wa)
        pb, _ = run_w(wb)
        if pall is not None:
            out["linearity_rel_l2"] = float((pall - pa - pb).norm() / pall.norm())
            out["linearity_ok"] = out["linearity_rel_l2"] <= 1e-10
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
