"""Benchmark: dirty-image throughput of the B200 w-stacking hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the hot path over one batch of synthetic input:
prepare -> bucket -> grid -> per-plane inverse FFT -> w correction + stack ->
dirty image (pipeline.py:95-152). At N=1 the workload is BASELINE config 2
(10M records, 2048x2048x32, Gaussian support 7, FP64, 1 GPU). Inputs
(360 MB) and grid (2 GiB) are larger than L2, so no explicit flush is needed.

value  : records imaged per second over the whole step (Mvis/s), inputs
         resident in HBM, CUDA events on the launching stream, max over ranks.
e2e    : the same through the public host-buffer API (wsb_image): pinned host
         arrays in, host image out, copies inside the timed region.
roofline: algorithmic bytes / measured time of the dominant kernel against
         the measured HBM copy bandwidth (MEASURED_PEAKS.json).
cpu_baseline / --impl reference: the CPU oracle (a NumPy restatement of the
         reference algorithm, oracle/) imaging full cfg2 batches on all host
         cores, measured (N > 1: gridding scaled to the job's records).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG2 = dict(n_vis=10_000_000, n_u=2048, n_v=2048, n_w=32, cell=2e-4, w_max=1000.0,
            kind="gaussian", S=3, shape=1.0, seed=1)
SOURCES = ((0.02, -0.015, 2.0), (0.0, 0.0, 1.0), (-0.05, 0.03, 0.5))


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def synthetic(cfg, n=None, seed=None):
    """generate_synthetic (visdata.py:384-434) restated: PCG64 uniform uvw,
    exact point-source visibilities, unit weights, time-sorted."""
    n = cfg["n_vis"] if n is None else n
    rng = np.random.default_rng(cfg["seed"] if seed is None else seed)
    u = rng.random(n)
    v = rng.random(n)
    w = rng.random(n)
    t = (np.arange(n, dtype=np.uint64) * 8 // max(n, 1)).astype(np.uint32)
    cell = cfg["cell"]
    un, vn, wn = u / cell, v / cell, w * cfg["w_max"]
    val = np.zeros(n, np.complex128)
    for l, m, f in SOURCES:
        nn = np.sqrt(1.0 - l * l - m * m)
        val += (f / nn) * np.exp(-2j * np.pi * (un * l + vn * m + wn * (nn - 1.0)))
    vis = val.astype(np.complex64)[:, None]
    wt = np.ones((n, 1), np.float32)
    return u, v, w, t, vis, wt


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class NvmlClockSampler:
    """SM clock and throttle reasons sampled through NVML every 5 ms during
    the timed region (nvidia-smi's 100 ms period gives one sample of a
    0.1 s region). Same interface as ClockSampler."""

    PERIOD = 0.005
    BITS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
            ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, dev):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        idx = dev.index if hasattr(dev, "index") and dev.index is not None else int(dev)
        try:   # the CUDA device's PCI address (CUDA_VISIBLE_DEVICES may renumber)
            props = torch.cuda.get_device_properties(idx)
            bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
        self.reasons_fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(pynvml, "nvmlDeviceGetCurrentClocksThrottleReasons")
        self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)    # (raise here, not in the thread)
        self.reasons_fn(self.h)
        self.samples = []
        self.stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = self.reasons_fn(self.h)
                self.samples.append((time.perf_counter(), float(sm), int(rs)))
            except Exception:
                pass
            time.sleep(self.PERIOD)

    def __enter__(self):
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()
        return self

    def mark(self, which: str):
        setattr(self, "t_" + which, time.perf_counter())

    def __exit__(self, *exc):
        self.stop.set()
        self.thread.join(timeout=2)

    def summary(self):
        t0, t1 = getattr(self, "t_start", -1e18), getattr(self, "t_end", 1e18)
        inside = [x for x in self.samples if t0 <= x[0] <= t1]
        if not inside and self.samples:
            inside = [min(self.samples, key=lambda x: abs(x[0] - t1))]
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": self.mx, "reasons": [], "samples": 0, "source": "nvml"}
        reasons = sorted({nm for _, _, rs in inside for nm, bit in self.BITS if rs & bit})
        return {"sm_mhz": float(np.median([x[1] for x in inside])), "sm_max_mhz": self.mx,
                "reasons": reasons, "samples": len(inside), "source": "nvml, 5 ms period"}


def clock_sampler(dev):
    """NVML sampler when pynvml can see the device, else nvidia-smi."""
    try:
        return NvmlClockSampler(dev)
    except Exception as e:
        log(f"NVML clock sampler unavailable ({type(e).__name__}: {e}); nvidia-smi at 100 ms")
        return ClockSampler(dev.index if hasattr(dev, "index") else int(dev))


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self, which: str):
        setattr(self, "t_" + which, time.perf_counter())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        t0, t1 = getattr(self, "t_start", -1e18), getattr(self, "t_end", 1e18)
        inside = [ln for t, ln in self.lines if t0 <= t <= t1 + 0.1]
        if not inside and self.lines:  # timed region shorter than the sampling period
            inside = [min(self.lines, key=lambda x: abs(x[0] - t1))[1]]
        for ln in inside:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def kernel_table(cfg, ms, ws=1):
    """Algorithmic bytes per launch group against the
    measured per-kernel times ms = [prepare, bucket, grid, fft_rows, fft_cols, finish]
    of one rank (which holds 1/ws of the mesh)."""
    N = cfg["n_vis"]
    cells = cfg["n_u"] * cfg["n_v"] * cfg["n_w"] // ws
    pix = cfg["n_u"] * cfg["n_v"] // ws
    groups = {
        # K1+K2: vis read once (36 B) + grid written once (16 B/cell)
        "gridder(K1+K2)": (N * 36 + cells * 16, ms[0] + ms[1] + ms[2]),
        "grid(K2)": (cells * 16, ms[2]),
        "fft_rows(K3a)": (cells * 32, ms[3]),
        # column FFT + w correction + stacking: planes read once, image written once
        "fft_cols_stack(K3b+K4)": (cells * 16 + pix * 8, ms[4]),
    }
    return groups


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2504_00959_b200 as W

    ws, rank, local = dist_env()
    if ws > 1:
        from paper_2504_00959_b200 import distributed as WD
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)
    cfg = dict(CFG2)
    spec = W.GridSpec(cfg["n_u"], cfg["n_v"], cfg["n_w"], cfg["cell"], w_max_native=cfg["w_max"])
    # multi-GPU decomposition (distributed.image_distributed's "auto" rule)
    decomp = args.decomp if args.decomp != "auto" else ("planes" if ws <= cfg["n_w"] else "slabs")
    kern = W.KernelSpec(cfg["kind"], cfg["S"], cfg["shape"])

    # weak scaling: every rank holds its own 10M-record time partition
    t0 = time.perf_counter()
    u, v, w, t, vis, wt = synthetic(cfg, seed=cfg["seed"] + rank)
    log(f"[rank {rank}] synthetic {cfg['n_vis']} records in {time.perf_counter() - t0:.1f}s")
    du, dv, dw = (torch.from_numpy(a).to(dev) for a in (u, v, w))
    dvis = torch.from_numpy(vis).to(dev)
    dwt = torch.from_numpy(wt).to(dev)
    img = torch.empty((cfg["n_v"], cfg["n_u"]), dtype=torch.float64, device=dev)

    def step():
        if ws > 1:
            return WD.image_distributed(du, dv, dw, dvis, dwt, spec, kern, to_host=False,
                                        decomposition=decomp)
        return W.image_device(du, dv, dw, dvis, dwt, spec, kern, image_out=img)

    clk = clock_sampler(dev).__enter__()   # sampling runs through warm-up and timing
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    per_kernel = np.zeros(6)
    launches = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.mark("start")
    launches0 = W.last_timings(dev)[1]   # cumulative counter of the multi-stage path
    ev0.record(stream)
    for _ in range(args.steps):
        step()
        if ws == 1:
            ms, nl = W.last_timings(dev)
            per_kernel += np.array(ms)
            launches += nl
    ev1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        launches = W.last_timings(dev)[1] - launches0
    clk.mark("end")
    clk.__exit__(None, None, None)
    if ws > 1:
        dist.barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    if ws > 1:
        tt = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms = float(tt.item())
    ms_step = elapsed_ms / args.steps
    total_vis = cfg["n_vis"] * ws
    value = total_vis / (ms_step / 1e3) / 1e6

    # multi-GPU: per-stage times of the compute stream from a few extra
    # (untimed) steps with stage events; the bucket / sweep split comes from
    # the library's own events around the gridder
    stages = None
    if ws > 1:
        acc = {}
        n_st = 3
        for _ in range(n_st):
            tm = {}
            WD.image_distributed(du, dv, dw, dvis, dwt, spec, kern, to_host=False, timings=tm,
                                 decomposition=decomp)
            for k_, v_ in tm.items():
                acc[k_] = acc.get(k_, 0.0) + v_ / n_st
        stages = {k_: round(v_, 4) for k_, v_ in acc.items()}
        per_kernel = np.array([acc.get("prepare", 0.0), acc.get("bucket", 0.0), acc.get("sweep", 0.0),
                               acc.get("rows", 0.0), acc.get("cols", 0.0), 0.0]) * args.steps

    # energy to solution: NVML (+ RAPL) over a >= 1 s window of the same step
    energy = None
    try:
        from paper_2504_00959_b200.energy import NvmlRaplMeter
        meter = NvmlRaplMeter(devices=[dev.index], host=(rank == 0))
        n_en = max(args.steps, int(1.0 / max(ms_step / 1e3, 1e-4)) + 1)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        meter.start()
        t0 = time.perf_counter()
        for _ in range(n_en):
            step()
        torch.cuda.synchronize()
        win = time.perf_counter() - t0
        j = meter.joules({"window": win}, "default")
        gj = torch.tensor([j["gpu"]], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(gj)
        host = j.get("host")
        host_src = "RAPL package counters (rank 0 host)"
        if host is None:
            from paper_2504_00959_b200.energy import ModelledHostMeter
            hm = ModelledHostMeter()
            host = hm.joules({"window": win})["window"]
            host_src = hm.source + "; RAPL unreadable on this host"
        energy = {"gpu_joules_per_step": round(float(gj.item()) / n_en, 4),
                  "host_joules_per_step": round(host / n_en, 4),
                  "window_s": round(win, 3), "steps": n_en,
                  "source": f"GPU: NVML total energy (all GPUs); host: {host_src}"}
    except Exception as exc:  # NVML missing or not permitted: report, do not fail the bench
        energy = {"unavailable": f"{type(exc).__name__}: {exc}"}

    # end-to-end through the host-buffer C ABI (pinned inputs, host image out)
    e2e = None
    if ws > 1:
        # every rank: its pinned host records -> device -> distributed image ->
        # host image on the root; wall time per step, max over ranks
        pin = [torch.from_numpy(a).pin_memory().numpy() for a in (u, v, w, vis, wt)]
        batch = tuple(pin)
        for _r in WD.image_distributed_stream([batch] * 4, spec, kern, decomposition=decomp):
            pass
        torch.cuda.synchronize()
        n_e2e = max(4, min(args.steps, 12))
        dist.barrier()
        t0 = time.perf_counter()
        for res, _ in WD.image_distributed_stream([batch] * n_e2e, spec, kern,
                                                  decomposition=decomp):
            pass
        torch.cuda.synchronize()
        e2e_s = torch.tensor([(time.perf_counter() - t0) / n_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e_s = float(e2e_s.item())
        h2d = sum(a.nbytes for a in (u, v, w, vis, wt)) * ws
        e2e = {"value": round(total_vis / e2e_s / 1e6, 2), "unit": "Mvis/s",
               "ms_per_step": round(e2e_s * 1e3, 3), "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(cfg["n_u"] * cfg["n_v"] * 8),
               "steps": n_e2e,
               "api": "paper_2504_00959_b200.distributed.image_distributed_stream (pinned host "
                      "batches on every rank -> host image on the root)"}
    if ws == 1:
        pin = [torch.from_numpy(a).pin_memory() for a in (u, v, w, vis, wt)]
        pu, pv, pw, pvis, pwt = (p.numpy() for p in pin)
        # warm-up in the timed loop's own pattern (the previous image is still
        # held when the next call allocates its page-locked result), so both
        # recycled host buffers exist before timing
        for _ in range(3):
            res, _ = W.image(pu, pv, pw, None, pvis, pwt, spec, kern, device=dev.index)
        torch.cuda.synchronize()
        n_e2e = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            res, _ = W.image(pu, pv, pw, None, pvis, pwt, spec, kern, device=dev.index)
        single_s = (time.perf_counter() - t0) / n_e2e
        # the streaming entry point: one image per batch, every batch copied
        # in and its image copied out, copies overlapped with the previous /
        # next batch's device work (fill and drain included in the time)
        n_st = max(4, min(args.steps, 12))
        batch = (pu, pv, pw, pvis, pwt)
        # warm-up in the timed loop's own pattern: the caller holds image i-1
        # while image i is pending and i+1 is produced, so three page-locked
        # images must exist before timing (pinning inside the loop costs ms)
        for _img in W.image_stream([batch] * 4, spec, kern, device=dev.index):
            pass
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for img_s, _d in W.image_stream([batch] * n_st, spec, kern, device=dev.index):
            pass
        e2e_s = (time.perf_counter() - t0) / n_st
        h2d = sum(a.nbytes for a in (u, v, w, vis, wt))
        e2e = {"value": round(cfg["n_vis"] / e2e_s / 1e6, 2), "unit": "Mvis/s",
               "ms_per_step": round(e2e_s * 1e3, 3), "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(img_s.pixels.nbytes), "steps": n_st,
               "api": "paper_2504_00959_b200.image_stream (pinned host batches -> host images)",
               "single_call": {"value": round(cfg["n_vis"] / single_s / 1e6, 2),
                               "ms_per_step": round(single_s * 1e3, 3),
                               "api": "paper_2504_00959_b200.image -> wsb_image (include/wsb.h)"}}

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    per_kernel /= args.steps
    peak, peak_kind = measured_peaks()
    groups = kernel_table(cfg, per_kernel, ws)
    if stages and "fft" in stages and not per_kernel[3] and not per_kernel[4]:
        # w-plane decomposition: the row and column passes of the local planes
        # are timed together as one "fft" stage (its plane ranges interleave
        # the two kernels); report them as one group instead of two zeros
        b_rows, _ = groups.pop("fft_rows(K3a)")
        b_cols, _ = groups.pop("fft_cols_stack(K3b+K4)")
        groups["fft_rows+cols_stack(K3+K4)"] = (b_rows + b_cols, stages["fft"])
    kernels = {}
    for name, (bytes_, t_ms) in groups.items():
        ach = bytes_ / (t_ms / 1e3) / 1e9 if t_ms > 0 else 0.0
        kernels[name] = {"ms": round(t_ms, 4), "algorithmic_bytes": int(bytes_),
                         "achieved_gbs": round(ach, 1), "frac": round(ach / peak, 3)}
    dom = max((k for k in kernels if k != "gridder(K1+K2)"), key=lambda k: kernels[k]["ms"])
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists() and ws == 1:   # captured on the 1-GPU step (one rank's share differs)
        traffic = json.loads(tf.read_text()).get(dom)
    roof = {"kernel": dom, "bound": "hbm", "achieved": kernels[dom]["achieved_gbs"],
            "peak": peak, "peak_source": peak_kind, "unit": "GB/s", "frac": kernels[dom]["frac"],
            "traffic": traffic,
            "bytes_per_launch": kernels[dom]["algorithmic_bytes"],
            "note": "achieved = algorithmic bytes / CUDA-event time of the kernel on its stream"}
    gridder = kernels["gridder(K1+K2)"]
    out = {
        "metric": "Mvis/s imaged (bucket+grid+FFT+w-stack, dirty image out)",
        "value": round(value, 2), "unit": "Mvis/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2: synthetic 10M visibilities per GPU, 2048x2048 grid, "
                               "32 w-planes, Gaussian support 7 (S=3, sigma=1), single channel, FP64",
                   "records_per_gpu": cfg["n_vis"], "n_u": cfg["n_u"], "n_v": cfg["n_v"],
                   "n_w": cfg["n_w"], "cell_size_lm": cfg["cell"], "w_max_native": cfg["w_max"],
                   "parallelism": ((f"v-slab x{ws}" if decomp == "slabs" else f"w-plane ranges x{ws}")
                                   if ws > 1 else "single GPU"),
                   "l2": "inputs 360 MB and grid 2 GiB exceed the 126 MB L2; no flush"},
        "gridding_mvis_s": round(cfg["n_vis"] / (gridder["ms"] / 1e3) / 1e6, 1) if gridder["ms"] else None,
        "roofline": roof,
        "kernels": kernels,
        "stages_ms": stages,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "e2e": e2e,
        "energy": energy,
    }
    if ws == 1 and not args.no_cfg3:
        try:
            out["cfg3"] = bench_cfg3(W, peak)
        except Exception as exc:   # report, do not fail the headline line
            out["cfg3"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
    if ws == 1 and not args.no_cpu_baseline:
        cb = out["cpu_baseline"] = cpu_baseline(cfg)
        # green productivity, Eq. 4 (metrics.py:200-207): reference run = the
        # CPU image (host energy), test run = the GPU step (NVML + host)
        if energy and energy.get("host_joules_per_step") is not None:
            from paper_2504_00959_b200.energy import green_productivity
            e_gpu = energy["gpu_joules_per_step"] + energy["host_joules_per_step"]
            out["green_productivity"] = {
                "value": round(green_productivity(cb["seconds_per_image"],
                                                  cb["host_joules_per_image"],
                                                  ms_step / 1e3, e_gpu), 1),
                "alpha": 1.0,
                "ref": {"seconds": cb["seconds_per_image"], "joules": cb["host_joules_per_image"],
                        "energy": cb["host_energy_source"]},
                "test": {"seconds": round(ms_step / 1e3, 6), "joules": round(e_gpu, 4),
                         "energy": energy["source"]},
                "formula": "(t_ref / t_test) / (alpha * E_test / E_ref), metrics.py:200-207"}
        else:
            out["green_productivity"] = None
    if ws > 1:
        dist.destroy_process_group()
    print(json.dumps(out), flush=True)


def bench_cfg3(W, peak, steps=5):
    """The north-star configuration on this GPU (BASELINE config 3): 100M
    LOFAR-like track records (tools/lofar.py, generated on the device),
    4096^2 x 64, Gaussian support 7, FP64. Device-resident inputs, CUDA
    events, per-kernel fractions of the HBM roofline against the SURVEY 8(d)
    algorithmic bytes, and the size-independent parity property the full
    size allows (linearity over complementary record halves; the
    slab-restricted oracle check of the densest rows is
    tests/test_gpu_scale.py::test_cfg3_densest_rows_vs_slab_restricted_oracle)."""
    import torch
    sys.path.insert(0, str(ROOT / "tools"))
    from lofar import tracks
    n, nu, nw, cell = 100_000_000, 4096, 64, 1e-4
    dev = torch.device("cuda", 0)
    u, v, w, t, vis, wt = tracks(n, cell, device=dev)
    spec = W.GridSpec(nu, nu, nw, cell, w_max_native=1000.0)
    kern = W.KernelSpec.gaussian(3, 1.0)
    for _ in range(2):
        W.image_device(u, v, w, vis, wt, spec, kern)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms_k = np.zeros(6)
    e0.record(stream)
    for _ in range(steps):
        W.image_device(u, v, w, vis, wt, spec, kern)
        ms_k += np.array(W.last_timings(dev)[0])
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ms_k /= steps
    cfg = dict(n_vis=n, n_u=nu, n_v=nu, n_w=nw)
    kernels = {}
    for name, (b, t_ms) in kernel_table(cfg, ms_k).items():
        ach = b / (t_ms / 1e3) / 1e9 if t_ms > 0 else 0.0
        kernels[name] = {"ms": round(t_ms, 3), "algorithmic_bytes": int(b),
                         "floor_ms": round(b / (peak * 1e9) * 1e3, 3),
                         "achieved_gbs": round(ach, 1), "frac": round(ach / peak, 3)}
    # linearity: image(all) = image(A) + image(B), complementary weight halves
    g = torch.Generator(device=dev).manual_seed(7)
    mask = torch.rand(wt.shape, generator=g, device=dev) < 0.5
    pall, _ = W.image_device(u, v, w, vis, wt, spec, kern)
    pall = pall.clone()
    pa, _ = W.image_device(u, v, w, vis, torch.where(mask, wt, torch.zeros_like(wt)), spec, kern)
    pa = pa.clone()
    pb, d = W.image_device(u, v, w, vis, torch.where(mask, torch.zeros_like(wt), wt), spec, kern)
    lin = float((pall - pa - pb).norm() / pall.norm())
    return {"workload": "cfg3: 100M LOFAR-like track records (62 stations, tools/lofar.py), "
                        "4096x4096 grid, 64 w-planes, Gaussian support 7, FP64, 1 GPU",
            "value": round(n / (ms / 1e3) / 1e6, 1), "unit": "Mvis/s", "ms_per_step": round(ms, 3),
            "steps": steps, "grid_updates": int(d["grid_updates"]), "kernels": kernels,
            "parity": {"linearity_rel_l2": lin, "ok": lin <= 1e-10,
                       "oracle": "tests/test_gpu_scale.py::test_cfg3_densest_rows_vs_slab_restricted_oracle"}}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _cpu_model():
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_meter():
    """RAPL package counters when readable, else the labelled power model
    (energy.ModelledHostMeter). Returns (meter, source, measured?)."""
    from paper_2504_00959_b200 import energy as E
    try:
        m = E.NvmlRaplMeter(devices=[], host=True)
        if m.host_available:
            return m, "RAPL package counters", True
    except Exception:
        pass
    m = E.ModelledHostMeter()
    return m, m.source, False


class CpuImage:
    """The reference algorithm (oracle port: NumPy restatement of
    prepare_chunk / exchange / tap-major np.add.at gridding / FFT / w screen /
    stack, oracle/wstack_oracle.py) imaging ONE full batch of records on the
    host cores: row-block gridding threads (the reference's deterministic
    threaded mode, gridder.py:206-221) and plane-parallel transforms.
    Inputs are generated before the timed call."""

    def __init__(self, cfg, n_records, threads, seed):
        from oracle import wstack_oracle as O
        self.O = O
        self.cfg = cfg
        self.threads = threads
        self.n = n_records
        self.data = synthetic(cfg, n=n_records, seed=seed)

    def run(self):
        O, c = self.O, self.cfg
        u, v, w, t, vis, wt = self.data
        kind = O.KIND_GAUSSIAN if c["kind"] == "gaussian" else O.KIND_KAISER_BESSEL
        t0 = time.perf_counter()
        r = O.image(u, v, w, t, vis, wt, c["n_u"], c["n_v"], c["n_w"], c["cell"], 0.0, c["w_max"],
                    kind, c["S"], c["shape"], threads=self.threads)
        return time.perf_counter() - t0, r


def cpu_baseline(cfg):
    """One full cfg2 image (10M records, 2048^2 x 32) by the oracle port on
    all host cores, measured (no extrapolation), with host energy."""
    threads = cpu_cores()
    job = CpuImage(cfg, cfg["n_vis"], threads, cfg["seed"] + 1000)
    meter, src, measured = host_meter()
    meter.start()
    secs, r = job.run()
    host_j = meter.joules({"image": secs}, "default")
    host_j = host_j.get("host", host_j.get("image"))
    return {"value": round(cfg["n_vis"] / secs / 1e6, 4), "unit": "Mvis/s", "cores": threads,
            "seconds_per_image": round(secs, 2), "host_joules_per_image": round(host_j, 1),
            "host_energy_source": src, "host_energy_measured": measured,
            "kind": "port",
            "sample": (f"one full cfg2 image measured (no scaling): {cfg['n_vis']} records "
                       f"gridded on the 2048x2048x32 mesh + 32 plane transforms / w screens / "
                       f"stack, oracle port, {threads} threads "
                       f"(grid_updates {r['grid_updates']})"),
            "cpu": _cpu_model()}


def run_reference(args):
    """The reference arm: the reference's algorithm (oracle port, oracle/) on
    the host cores, rank 0 only, same metric and configuration as our arm.

    N = 1: every timed step images the full cfg2 batch (10M records,
    2048^2 x 32): measured, nothing scaled; one untimed warm-up image.
    N > 1 (the job images N x 10M records on one mesh): each step grids a
    10M-record batch and transforms/stacks the full mesh, and the gridding
    time is scaled by N (gridding is linear in the records on a fixed mesh;
    the transforms do not depend on them) so the run stays within minutes."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = dict(CFG2)
    threads = cpu_cores()
    job = CpuImage(cfg, cfg["n_vis"], threads, cfg["seed"])
    n_warm = 1 if args.warmup > 0 else 0
    for _ in range(n_warm):
        job.run()
    times = []
    t_fft = None
    for _ in range(args.steps):
        secs, _r = job.run()
        if ws > 1:
            if t_fft is None:    # the mesh part of a step (transforms + stack), once
                from oracle import wstack_oracle as O
                g = np.zeros((cfg["n_w"], cfg["n_v"], cfg["n_u"]), np.complex128)
                t0 = time.perf_counter()
                O.image_from_grid(g, cfg["n_u"], cfg["n_v"], cfg["n_w"], cfg["cell"], 0.0,
                                  cfg["w_max"], threads)
                t_fft = time.perf_counter() - t0
                del g
            secs = t_fft + (secs - t_fft) * ws
        times.append(secs)
    s = float(np.mean(times))
    value = cfg["n_vis"] * ws / s / 1e6
    if ws == 1:
        sample = (f"per step: one full cfg2 image ({cfg['n_vis']} records, 2048x2048x32), "
                  f"measured; {n_warm} untimed warm-up image")
    else:
        sample = (f"per step: {cfg['n_vis']} records gridded + the full 2048x2048x32 mesh "
                  f"transformed/stacked, measured; gridding scaled x{ws} to the job's "
                  f"{ws} x {cfg['n_vis']} records")
    out = {"impl": "reference", "metric": "Mvis/s imaged (bucket+grid+FFT+w-stack, dirty image out)",
           "value": round(value, 4), "unit": "Mvis/s", "n_gpus": ws, "steps": args.steps,
           "warmup": n_warm, "ms_per_step": round(s * 1e3, 1), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "cfg2: synthetic 10M visibilities per GPU, 2048x2048 grid, "
                                  "32 w-planes, Gaussian support 7 (S=3, sigma=1), single channel, "
                                  "FP64", "records_total": cfg["n_vis"] * ws},
           "cpu_baseline": {"value": round(value, 4), "unit": "Mvis/s", "cores": threads,
                            "kind": "port", "sample": sample, "cpu": _cpu_model()},
           "e2e": {"value": round(value, 4), "unit": "Mvis/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cfg3", action="store_true", help="skip the cfg3 (north-star) object")
    ap.add_argument("--decomp", choices=["auto", "slabs", "planes"], default="auto",
                    help="multi-GPU decomposition: v-slabs (grid transpose) or w-plane ranges "
                         "(partial-stack reduce)")
    args = ap.parse_args()
    # stdout carries exactly the one JSON line: native libraries (NCCL prints
    # its version banner at communicator init) write to fd 1 directly, so fd 1
    # is pointed at stderr and Python's stdout keeps a private copy of it
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(json_fd, "w", buffering=1)
    if args.warmup < 3 and args.impl == "ours":
        log("note: warmup < 3 does not meet the timing rules")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
