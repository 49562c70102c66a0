"""Host-side mirror of the reference imaging API on the B200 kernels.

The reference's drop-in boundary is Python:
``pipeline.run_pipeline`` (pipeline.py:61-191) and the finer hooks
``gridder.grid_sector`` (gridder.py:186-259) and ``gridder.grid_all``
(gridder.py:262-294). This module keeps those names, argument meanings and
error behaviour (ValueError for invalid specs and inputs) and routes every
numeric step through libwsb.so. There is no CPU compute path.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import struct
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _lib as L

KERNEL_KINDS = ("gaussian", "kaiser_bessel")
DEFAULT_KB_BETA_PER_SUPPORT = 2.34
OPS_COLUMNS = ("records", "grid_updates", "exchange_bytes", "reduce_bytes", "fft_bytes",
               "reduce_messages", "stack_pixels")


# ---------------------------------------------------------------------------
# specs (mesh.py:59-112, gridder.py:47-72)
# ---------------------------------------------------------------------------

_C_STRUCTS: dict = {}   # GridSpec / KernelSpec -> their ctypes struct (the C side only reads it)


def _is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


@dataclass(frozen=True)
class GridSpec:
    n_u: int
    n_v: int
    n_w: int
    cell_size_lm: float
    w_min: float = 0.0
    w_max: float = 1.0
    w_min_native: float = 0.0
    w_max_native: float = 0.0

    def __post_init__(self):
        if self.n_u < 2 or not _is_pow2(self.n_u):
            raise ValueError(f"n_u must be a power of two >= 2, got {self.n_u}")
        if self.n_v < 2 or not _is_pow2(self.n_v):
            raise ValueError(f"n_v must be a power of two >= 2, got {self.n_v}")
        if self.n_w < 1:
            raise ValueError(f"n_w must be >= 1, got {self.n_w}")
        if self.cell_size_lm <= 0.0:
            raise ValueError("cell_size_lm must be positive")
        half_l = self.n_u * self.cell_size_lm / 2.0
        half_m = self.n_v * self.cell_size_lm / 2.0
        if half_l >= 1.0 or half_m >= 1.0 or half_l * half_l + half_m * half_m >= 1.0:
            raise ValueError("field of view too wide: corner pixels leave the unit disc")
        if self.w_min_native > self.w_max_native:
            raise ValueError("w_min_native must be <= w_max_native")

    def plane_w_native(self, k: int) -> float:
        if not (0 <= k < self.n_w):
            raise ValueError(f"plane {k} outside range(0, {self.n_w})")
        if self.n_w == 1:
            return 0.5 * (self.w_min_native + self.w_max_native)
        return self.w_min_native + (k / (self.n_w - 1)) * (self.w_max_native - self.w_min_native)

    def c_struct(self) -> L.WsbGrid:
        c = _C_STRUCTS.get(self)
        if c is None:   # (one ctypes struct per distinct spec)
            c = _C_STRUCTS[self] = L.grid_struct(self.n_u, self.n_v, self.n_w, self.cell_size_lm,
                                                 self.w_min_native, self.w_max_native)
        return c


@dataclass(frozen=True)
class KernelSpec:
    kind: str = "gaussian"
    half_support: int = 3
    shape_param: float = 1.0

    def __post_init__(self):
        if self.kind not in KERNEL_KINDS:
            raise ValueError(f"kernel kind must be one of {KERNEL_KINDS}, got {self.kind!r}")
        if self.half_support < 1:
            raise ValueError("half_support must be >= 1")
        if self.shape_param <= 0:
            raise ValueError("shape_param must be positive")

    @classmethod
    def gaussian(cls, half_support: int = 3, sigma: float = 1.0) -> "KernelSpec":
        return cls(kind="gaussian", half_support=half_support, shape_param=sigma)

    @classmethod
    def kaiser_bessel(cls, half_support: int = 3, beta: float | None = None) -> "KernelSpec":
        if beta is None:
            beta = DEFAULT_KB_BETA_PER_SUPPORT * half_support
        return cls(kind="kaiser_bessel", half_support=half_support, shape_param=beta)

    def c_struct(self) -> L.WsbKernel:
        c = _C_STRUCTS.get(self)
        if c is None:
            c = _C_STRUCTS[self] = L.kernel_struct(KERNEL_KINDS.index(self.kind), self.half_support,
                                                   self.shape_param)
        return c


def as_grid_spec(spec) -> GridSpec:
    """Accept our GridSpec or any object with the reference GridSpec fields."""
    if isinstance(spec, GridSpec):
        return spec
    return GridSpec(spec.n_u, spec.n_v, spec.n_w, spec.cell_size_lm,
                    getattr(spec, "w_min", 0.0), getattr(spec, "w_max", 1.0),
                    getattr(spec, "w_min_native", 0.0), getattr(spec, "w_max_native", 0.0))


def as_kernel_spec(k) -> KernelSpec:
    if isinstance(k, KernelSpec):
        return k
    return KernelSpec(k.kind, int(k.half_support), float(k.shape_param))


def partition_1d(n: int, parts: int, index: int):
    """mesh.py:34-45."""
    if parts < 1 or not (0 <= index < parts):
        raise ValueError(f"invalid partition index {index} of {parts}")
    q, r = divmod(n, parts)
    if index < r:
        return index * (q + 1), q + 1
    return r * (q + 1) + (index - r) * q, q


# ---------------------------------------------------------------------------
# results (transform.py:72-83, pipeline.py:28-38, metrics.py:67-101)
# ---------------------------------------------------------------------------

@dataclass
class FinalImage:
    spec: GridSpec
    pixels: np.ndarray
    imag_residual_norm: float = 0.0
    real_norm: float = 0.0


FREQ_LEVELS = ("default", "high", "medium", "low")   # metrics.py:53


class MeterError(Exception):
    """An energy meter cannot produce a measurement (metrics.py:62-63)."""


@dataclass
class RunRecord:
    """Per-phase wall times and joules of one run (metrics.py:67-101)."""

    label: str
    topology: object
    freq_level: str
    phase_times: dict
    energy_joules: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.freq_level not in FREQ_LEVELS:
            raise ValueError(f"freq_level must be one of {FREQ_LEVELS}")
        if "total" not in self.phase_times:
            raise ValueError("phase_times must include 'total'")
        for name, value in {**self.phase_times, **self.energy_joules}.items():
            if value < 0:
                raise ValueError(f"negative value for {name}: {value}")
        parts = sum(v for k, v in self.phase_times.items() if k != "total")
        if self.phase_times["total"] < parts - 1e-9:
            raise ValueError("total time smaller than the sum of its phases")

    @property
    def n_nodes(self) -> int:
        return self.topology.n_nodes if self.topology else 1

    @property
    def total_seconds(self) -> float:
        return self.phase_times["total"]

    @property
    def total_joules(self) -> float:
        if "total" not in self.energy_joules:
            raise MeterError(f"run {self.label!r} carries no total energy")
        return self.energy_joules["total"]


@dataclass
class PipelineResult:
    run: RunRecord
    image: FinalImage
    log: object
    ops: dict
    paths: dict = field(default_factory=dict)

    @property
    def image_sha256(self) -> str:
        return hashlib.sha256(self.image.pixels.astype("<f8").tobytes()).hexdigest()


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------

def _device_index(device) -> int:
    if device is None:
        return torch.cuda.current_device()
    if isinstance(device, torch.device):
        return device.index if device.index is not None else torch.cuda.current_device()
    if isinstance(device, str):
        return torch.device(device).index or 0
    return int(device)


def _require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2504_00959_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU path")


def context(device=None) -> L.Context:
    _require_cuda()
    dev = _device_index(device)
    ctx = L.Context.get(dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    if getattr(ctx, "_bound", None) != stream:     # (rebinding costs a C call per image)
        with torch.cuda.device(dev):
            ctx.bind_stream(stream)
        ctx._bound = stream
    return ctx


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _to_dev(a, dtype, dev) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        if a.dtype == dtype and a.device == dev and a.is_contiguous():
            return a                                  # (already in place: no dispatch)
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)


def _cols2d(a, n: int):
    """(n,) or (n, n_chan) -> (n, n_chan); keeps n_chan for empty inputs."""
    if a.ndim == 1:
        return a.reshape(n, 1)
    return a.reshape(n, a.shape[-1] if n == 0 else -1)


def _vis_f32(vis, n: int, dev) -> tuple[torch.Tensor, int]:
    """complex64 (n, n_chan) -> float32 (n, n_chan, 2) interleaved, on device."""
    if isinstance(vis, torch.Tensor):
        if (vis.dtype == torch.float32 and vis.device == dev and vis.dim() == 3 and vis.shape[0] == n
                and vis.shape[2] == 2 and vis.is_contiguous()):
            return vis, vis.shape[1]                  # (already interleaved f32 on the device)
        t = vis.to(dev)
        if t.is_complex():
            t = torch.view_as_real(_cols2d(t.to(torch.complex64), n).contiguous())
        t = t.reshape(n, -1, 2).to(torch.float32).contiguous()
        return t, t.shape[1]
    a = np.ascontiguousarray(_cols2d(np.asarray(vis), n), dtype=np.complex64)
    return torch.from_numpy(a.view(np.float32).reshape(n, -1, 2)).to(dev), a.shape[1]


# ---------------------------------------------------------------------------
# stages (device tensors)
# ---------------------------------------------------------------------------

def prepare_device(u, v, w, vis, weight, spec: GridSpec, device=None):
    """prepare_chunk (comms.py:477-492) on the GPU.

    Returns (rec f64 [n, 4] = (gu, gv, Re value, Im value), plane int32 [n])."""
    spec = as_grid_spec(spec)
    ctx = context(device)
    dev = torch.device("cuda", ctx.device)
    u = _to_dev(u, torch.float64, dev)
    n = u.numel()
    v = _to_dev(v, torch.float64, dev)
    w = _to_dev(w, torch.float64, dev)
    visf, n_chan = _vis_f32(vis, n, dev)
    wt = _to_dev(_cols2d(weight if isinstance(weight, torch.Tensor) else np.asarray(weight), n),
                 torch.float32, dev)
    if not (v.numel() == w.numel() == n and wt.shape == (n, n_chan)):
        raise ValueError("inconsistent column lengths")
    rec = torch.empty((max(n, 1), 4), dtype=torch.float64, device=dev)
    plane = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    g = spec.c_struct()
    L.check(L.lib().wsb_prepare(ctx.handle, C.byref(g), _ptr(u), _ptr(v), _ptr(w), _ptr(visf),
                                _ptr(wt), n, n_chan, _ptr(rec), _ptr(plane)))
    return rec[:n], plane[:n]


def grid_slab_device(rec: torch.Tensor, plane: torch.Tensor, spec: GridSpec, kern: KernelSpec,
                     v_start: int, v_count: int, out: torch.Tensor | None = None):
    """grid_sector (gridder.py:186-259) for one slab on the GPU. Returns
    (strip-layout grid, float64 [n_w, ceil(n_u/S), v_count, 2 (re, im), S]
    with S = WSB_STRIP, grid_updates)."""
    spec, kern = as_grid_spec(spec), as_kernel_spec(kern)
    ctx = context(rec.device)
    m = rec.shape[0]
    if out is None:
        sw = L.STRIP
        out = torch.empty((spec.n_w, (spec.n_u + sw - 1) // sw, v_count, 2, sw),
                          dtype=torch.float64, device=rec.device)
    upd = C.c_int64()
    g, k = spec.c_struct(), kern.c_struct()
    L.check(L.lib().wsb_grid_slab(ctx.handle, C.byref(g), C.byref(k), int(v_start), int(v_count),
                                  _ptr(rec.contiguous()), _ptr(plane.contiguous()), m, _ptr(out),
                                  C.byref(upd)))
    return out, int(upd.value)


def bucket_items_device(rec: torch.Tensor, plane: torch.Tensor, spec, half_support: int,
                        v_start: int, v_count: int):
    """The gridder's bucketing (K1) of prepared records, copied to the host:
    (keys u32, idx u32, off u32 [n_items + 1], item_bits) -- see
    wsb_bucket_items in include/wsb.h."""
    spec = as_grid_spec(spec)
    ctx = context(rec.device)
    m = rec.shape[0]
    g = spec.c_struct()
    ne, ni, ib = C.c_int64(), C.c_int64(), C.c_int32()
    L.check(L.lib().wsb_bucket_items(ctx.handle, C.byref(g), int(half_support), int(v_start),
                                     int(v_count), _ptr(rec.contiguous()),
                                     _ptr(plane.contiguous()), m, None, None, None,
                                     C.byref(ne), C.byref(ni), C.byref(ib)))
    keys = np.empty(max(ne.value, 1), np.uint32)
    idx = np.empty(max(ne.value, 1), np.uint32)
    off = np.empty(ni.value + 1, np.uint32)
    L.check(L.lib().wsb_bucket_items(ctx.handle, C.byref(g), int(half_support), int(v_start),
                                     int(v_count), _ptr(rec.contiguous()),
                                     _ptr(plane.contiguous()), m,
                                     keys.ctypes.data_as(C.c_void_p), idx.ctypes.data_as(C.c_void_p),
                                     off.ctypes.data_as(C.c_void_p), C.byref(ne), C.byref(ni),
                                     C.byref(ib)))
    return keys[:ne.value], idx[:ne.value], off, int(ib.value)


def unpack_grid_device(grid_p: torch.Tensor, spec: GridSpec, v_start: int, v_count: int,
                       rows: tuple | None = None):
    """Strip layout -> (n_w, v_count, n_u) complex128 without the checkerboard
    sign; ``rows`` = (row_lo, row_hi) (absolute rows inside the slab) keeps
    only those rows."""
    spec = as_grid_spec(spec)
    ctx = context(grid_p.device)
    r0, r1 = rows if rows is not None else (v_start, v_start + v_count)
    out = torch.empty((spec.n_w, r1 - r0, spec.n_u, 2), dtype=torch.float64, device=grid_p.device)
    g = spec.c_struct()
    L.check(L.lib().wsb_grid_unpack_rows(ctx.handle, C.byref(g), int(v_start), int(v_count),
                                         int(r0), int(r1), _ptr(grid_p), _ptr(out)))
    return torch.view_as_complex(out)


def image_device(u, v, w, vis, weight, spec, kern, image_out: torch.Tensor | None = None,
                 precision: int = 64):
    """Whole hot path on device-resident inputs (one GPU): returns
    (pixels f64 tensor (n_v, n_u), diag dict). precision=32 selects the FP32
    path (complex64 grid and transforms; within 1e-5 of the FP64 image)."""
    spec, kern = as_grid_spec(spec), as_kernel_spec(kern)
    dev = u.device if isinstance(u, torch.Tensor) and u.is_cuda else None
    ctx = context(dev)
    dev = torch.device("cuda", ctx.device)
    u = _to_dev(u, torch.float64, dev)
    n = u.numel()
    v = _to_dev(v, torch.float64, dev)
    w = _to_dev(w, torch.float64, dev)
    visf, n_chan = _vis_f32(vis, n, dev)
    wt = _to_dev(_cols2d(weight if isinstance(weight, torch.Tensor) else np.asarray(weight), n),
                 torch.float32, dev)
    if image_out is None:
        image_out = torch.empty((spec.n_v, spec.n_u), dtype=torch.float64, device=dev)
    d = L.WsbDiag()
    g, k = spec.c_struct(), kern.c_struct()
    lib = L.lib()
    if int(precision) == 64:   # (the context's default: no precision round trip)
        L.check(lib.wsb_image_device(ctx.handle, C.byref(g), C.byref(k), _ptr(u), _ptr(v), _ptr(w),
                                     _ptr(visf), _ptr(wt), n, n_chan, _ptr(image_out), C.byref(d)))
        return image_out, diag_dict(d)
    L.check(lib.wsb_ctx_set_precision(ctx.handle, int(precision)))
    try:
        L.check(lib.wsb_image_device(ctx.handle, C.byref(g), C.byref(k), _ptr(u), _ptr(v), _ptr(w),
                                     _ptr(visf), _ptr(wt), n, n_chan, _ptr(image_out), C.byref(d)))
    finally:
        lib.wsb_ctx_set_precision(ctx.handle, 64)
    return image_out, diag_dict(d)


def image_stream(batches, spec, kern, device: int = 0):
    """Dirty images of a stream of HOST record batches (one image per batch,
    e.g. successive time chunks of an observation), double-buffered: the
    host->device copy of batch i+1 and the device->host copy of image i-1
    run on their own streams (both PCIe directions) while batch i is imaged.
    Every batch still makes the full round trip; only the copies overlap the
    device work. Each batch is (u, v, w, vis, weight) as in ``image``;
    page-locked host arrays move at DMA speed. Yields (FinalImage, diag)."""
    spec, kern = as_grid_spec(spec), as_kernel_spec(kern)
    _require_cuda()
    dev = torch.device("cuda", int(device))
    ctx = context(dev)
    compute = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    sets = [None, None]            # device input buffers per slot
    imgs = [None, None]            # device images per slot
    done = [None, None]            # compute-finished event per slot
    read = [None, None]            # image-copied-out event per slot
    # page-locked images, recycled (across calls) once the caller drops them
    pool = _PINNED_POOLS.setdefault((spec.n_v, spec.n_u), [])

    def upload(i, b):
        u, v, w, vis, wt = b
        n = len(u)
        vis = _cols2d(np.asarray(vis, np.complex64), n)
        wt = _cols2d(np.asarray(wt, np.float32), n)
        host = [torch.from_numpy(np.ascontiguousarray(x)) for x in
                (np.asarray(u, np.float64), np.asarray(v, np.float64), np.asarray(w, np.float64),
                 vis.view(np.float32), wt)]
        slot = i % 2
        if sets[slot] is None or any(d.shape != h.shape for d, h in zip(sets[slot], host)):
            sets[slot] = [torch.empty(h.shape, dtype=h.dtype, device=dev) for h in host]
        with torch.cuda.stream(s_in):
            if done[slot] is not None:
                s_in.wait_event(done[slot])      # the slot's previous batch has been imaged
            for d, h in zip(sets[slot], host):
                d.copy_(h, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s_in)
        return ev, vis.shape[1], host

    it = iter(batches)
    nxt = next(it, None)
    if nxt is None:
        return
    staged = upload(0, nxt)
    pending = None                 # (event, pinned image, diag, slot) of the previous batch
    i = 0
    while staged is not None:
        ev, n_chan, _host = staged
        slot = i % 2
        nxt = next(it, None)
        compute.wait_event(ev)
        # the next upload is enqueued before this batch's (synchronising) call
        staged_next = upload(i + 1, nxt) if nxt is not None else None
        u, v, w, visf, wt = sets[slot]
        n = u.numel()
        if imgs[slot] is None:
            imgs[slot] = torch.empty((spec.n_v, spec.n_u), dtype=torch.float64, device=dev)
        if read[slot] is not None:
            compute.wait_event(read[slot])       # image of batch i-2 has left the device
        d = L.WsbDiag()
        g, k = spec.c_struct(), kern.c_struct()
        L.check(L.lib().wsb_image_device(ctx.handle, C.byref(g), C.byref(k), _ptr(u), _ptr(v),
                                         _ptr(w), _ptr(visf), _ptr(wt), n, n_chan,
                                         _ptr(imgs[slot]), C.byref(d)))
        done[slot] = torch.cuda.Event()
        done[slot].record(compute)
        # page-locked image from torch's caching host allocator (recycled
        # once the caller drops an image: no re-pinning in steady state); the
        # yielded pixels are that buffer itself, no host copy
        out = _pinned_image(pool, spec)
        with torch.cuda.stream(s_out):
            s_out.wait_event(done[slot])
            out.copy_(imgs[slot], non_blocking=True)
            oev = torch.cuda.Event()
            oev.record(s_out)
        read[slot] = oev
        if pending is not None:
            pev, pout, pd = pending
            pev.synchronize()
            yield (FinalImage(spec, pout.numpy(), pd.imag_residual_norm, pd.real_norm),
                   diag_dict(pd))
        pending = (oev, out, d)
        staged = staged_next
        i += 1
    pev, pout, pd = pending
    pev.synchronize()
    yield FinalImage(spec, pout.numpy(), pd.imag_residual_norm, pd.real_norm), diag_dict(pd)


_PINNED_POOLS: dict = {}


_PINNED_POOL_CAP = 3   # page-locked images kept per shape (the stream holds <= 3 in flight)


def _pinned_image(pool: list, spec) -> torch.Tensor:
    """A page-locked (n_v, n_u) float64 tensor from ``pool``: one nobody else
    references any more (the yielded numpy view holds its tensor), else a new
    one -- pinning is slow, so steady state allocates nothing and the image
    is handed out without a host copy. The pool keeps at most
    _PINNED_POOL_CAP buffers per shape; a caller holding more images at once
    (e.g. ``list(image_stream(...))``) gets un-pooled buffers that go back to
    torch's host allocator when dropped."""
    import sys
    for t in pool:
        # references: the pool list, the loop variable, getrefcount's argument
        if sys.getrefcount(t) <= 3:
            return t
    t = torch.empty((spec.n_v, spec.n_u), dtype=torch.float64, pin_memory=True)
    if len(pool) < _PINNED_POOL_CAP:
        pool.append(t)
    return t


def diag_dict(d: L.WsbDiag) -> dict:
    return {"imag_residual_norm": d.imag_residual_norm, "real_norm": d.real_norm,
            "grid_updates": int(d.grid_updates), "records": int(d.records),
            "tile_entries": int(d.tile_entries), "phase_ms": list(d.phase_ms),
            "exchanged_records": int(d.exchanged_records),
            "gpu_joules": d.gpu_joules if d.gpu_joules >= 0 else None,
            "host_joules": d.host_joules if d.host_joules >= 0 else None}


def last_timings(device=None):
    ctx = context(device)
    ms = (C.c_double * 6)()
    n = C.c_int32()
    L.check(L.lib().wsb_last_timings(ctx.handle, ms, C.byref(n)))
    return list(ms), int(n.value)


# ---------------------------------------------------------------------------
# host-buffer entry (the C-ABI drop-in, include/wsb.h wsb_image)
# ---------------------------------------------------------------------------

def image(u, v, w, time_index, vis, weight, spec, kern, device: int = 0,
          precision: int = 64, energy: bool = False) -> tuple[FinalImage, dict]:
    """Dirty image from HOST arrays through wsb_image (copies in and out are
    part of the call). Mirrors run_pipeline phases 2-5 (pipeline.py:95-152).
    ``energy`` reads the NVML / RAPL counters around the call into
    diag["gpu_joules"] / diag["host_joules"] (-1: unreadable)."""
    spec, kern = as_grid_spec(spec), as_kernel_spec(kern)
    _require_cuda()
    u = np.ascontiguousarray(u, np.float64)
    n = len(u)
    v = np.ascontiguousarray(v, np.float64)
    w = np.ascontiguousarray(w, np.float64)
    vis = np.ascontiguousarray(_cols2d(np.asarray(vis, np.complex64), n))
    weight = np.ascontiguousarray(_cols2d(np.asarray(weight, np.float32), n))
    if not (len(v) == len(w) == n and vis.shape == weight.shape):
        raise ValueError("inconsistent column lengths")
    # page-locked result buffer: the device->host copy runs at DMA speed
    # (a pageable destination costs ~10x on the 32 MB cfg2 image)
    out = torch.empty((spec.n_v, spec.n_u), dtype=torch.float64, pin_memory=True).numpy()
    d = L.WsbDiag()
    g, k = spec.c_struct(), kern.c_struct()
    ex = L.WsbExec(int(device), int(precision), 1, L.EXEC_ENERGY if energy else 0)
    ti = None if time_index is None else np.ascontiguousarray(time_index, np.uint32)
    vp = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)  # noqa: E731
    L.check(L.lib().wsb_image(C.byref(g), C.byref(k), C.byref(ex), vp(u), vp(v), vp(w), vp(ti),
                              vp(vis), vp(weight), n, vis.shape[1], vp(out), C.byref(d)))
    return FinalImage(spec, out, d.imag_residual_norm, d.real_norm), diag_dict(d)


# ---------------------------------------------------------------------------
# reference-compatible hooks
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SlabRange:
    """Rows [v_start, v_start + v_count) of one rank (mesh.py:113-126)."""
    rank: int
    v_start: int
    v_count: int

    @property
    def v_end(self) -> int:
        return self.v_start + self.v_count


def slab_of(spec, rank: int, n_ranks: int) -> SlabRange:
    """The v-slab of ``rank`` (mesh.py:152-159)."""
    if n_ranks < 1 or not (0 <= rank < n_ranks):
        raise ValueError(f"invalid rank {rank} of {n_ranks}")
    if n_ranks > spec.n_v:
        raise ValueError(f"n_ranks {n_ranks} exceeds n_v {spec.n_v}")
    v0, vc = partition_1d(spec.n_v, n_ranks, rank)
    return SlabRange(rank, v0, vc)


@dataclass
class ComplexGrid:
    """A slab of the mesh, (plane, v_row, u_col) complex128 (mesh.py:129-146)."""
    spec: object
    slab: SlabRange
    data: np.ndarray = None

    def __post_init__(self):
        shape = (self.spec.n_w, self.slab.v_count, self.spec.n_u)
        if self.data is None:
            self.data = np.zeros(shape, np.complex128)
        else:
            self.data = np.ascontiguousarray(self.data, np.complex128)
            if self.data.shape != shape:
                raise ValueError(f"grid data shape {self.data.shape} != {shape}")


@dataclass
class SectorBatch:
    """One slab's prepared records in (time_index, gindex) order
    (gridder.py:114-157); same validation: equal column lengths and every
    anchor row within the slab's +-halo_rows band."""
    slab: SlabRange
    gu: np.ndarray
    gv: np.ndarray
    plane: np.ndarray
    value: np.ndarray
    time_index: np.ndarray = None
    gindex: np.ndarray = None
    is_halo: np.ndarray = None
    halo_rows: int = 0

    def __post_init__(self):
        self.gu = np.ascontiguousarray(self.gu, np.float64)
        self.gv = np.ascontiguousarray(self.gv, np.float64)
        n = len(self.gu)
        self.plane = np.ascontiguousarray(self.plane, np.uint32)
        self.value = np.ascontiguousarray(self.value, np.complex128)
        self.time_index = (np.zeros(n, np.uint32) if self.time_index is None
                           else np.ascontiguousarray(self.time_index, np.uint32))
        self.gindex = (np.arange(n, dtype=np.uint64) if self.gindex is None
                       else np.ascontiguousarray(self.gindex, np.uint64))
        rows = np.floor(self.gv).astype(np.int64)
        if self.is_halo is None:
            self.is_halo = ~((rows >= self.slab.v_start) & (rows < self.slab.v_end))
        for a in (self.gv, self.plane, self.value, self.time_index, self.gindex, self.is_halo):
            if len(a) != n:
                raise ValueError("batch columns must share one length")
        if n and (rows.min() < self.slab.v_start - self.halo_rows - 1
                  or rows.max() > self.slab.v_end + self.halo_rows):
            raise ValueError("record outside slab+halo")

    def __len__(self) -> int:
        return len(self.gu)


def grid_sector(batch, kern, out, threads: int = 1, deterministic: bool = True) -> int:
    """gridder.grid_sector (gridder.py:186-259) on the GPU.

    ``batch`` carries gu, gv, plane, value (a SectorBatch, ours or the
    reference's); ``out`` has ``spec``, ``slab`` (v_start, v_count) and
    ``data`` (n_w, v_count, n_u) complex128, which is accumulated into like
    the reference does. Returns the number of cell updates.
    ``threads``/``deterministic`` are accepted for API parity: the GPU result
    is always deterministic (and bit-identical for any thread count)."""
    slab = out.slab
    if (slab.v_start, slab.v_count) != (batch.slab.v_start, batch.slab.v_count):
        raise ValueError("batch and output slab ranges differ")
    spec, kern = as_grid_spec(out.spec), as_kernel_spec(kern)
    n = len(batch.gu)
    if n == 0:
        return 0
    S = kern.half_support
    gv = np.asarray(batch.gv, np.float64)
    if np.any(gv + S < slab.v_start) or np.any(gv - S > slab.v_start + slab.v_count - 1):
        raise ValueError("record outside slab+halo")
    ctx = context()
    dev = torch.device("cuda", ctx.device)
    val = np.asarray(batch.value, np.complex128)
    rec = np.stack([np.asarray(batch.gu, np.float64), gv, val.real, val.imag], axis=1)
    rec_t = torch.from_numpy(np.ascontiguousarray(rec)).to(dev)
    plane_t = torch.from_numpy(np.asarray(batch.plane, np.int32)).to(dev)
    gp, upd = grid_slab_device(rec_t, plane_t, spec, kern, slab.v_start, slab.v_count)
    g = unpack_grid_device(gp, spec, slab.v_start, slab.v_count)
    out.data += g.cpu().numpy()
    return upd


def grid_all(per_rank_records, spec, kern, topo, strategy=None, log=None):
    """gridder.grid_all (gridder.py:262-294) for a virtual topology on one GPU:
    the ranks' record partitions (VisChunk-like: u, v, w, time_index, vis,
    weight; rank order = gindex order) go to the v-slab owners with the
    +-S halo (comms.py:495-547: records of a slab in (time_index, gindex)
    order), each slab is gridded (wsb_grid_slab) and returned as a
    ComplexGrid. The reduce is the identity after the exchange; the
    returned MessageLog holds the exchange and reduce messages the
    reference logs for ``topo`` (msglog.py). Bit-identical slabs for any
    rank count. Returns (slabs, log)."""
    from . import msglog
    spec, kern = as_grid_spec(spec), as_kernel_spec(kern)
    kind = getattr(strategy, "kind", "direct") if strategy is not None else "direct"
    R = int(topo.n_ranks)
    if len(per_rank_records) != R:
        raise ValueError(f"expected {R} record partitions, got {len(per_rank_records)}")
    S = kern.half_support
    ctx = context()
    dev = torch.device("cuda", ctx.device)
    lens = [len(c.u) for c in per_rank_records]
    cat = lambda name: np.concatenate([np.asarray(getattr(c, name)) for c in per_rank_records])  # noqa: E731
    u, v, w, t = cat("u"), cat("v"), cat("w"), cat("time_index").astype(np.uint32)
    vis = np.concatenate([_cols2d(np.asarray(c.vis), len(c.u)) for c in per_rank_records])
    wt = np.concatenate([_cols2d(np.asarray(c.weight), len(c.u)) for c in per_rank_records])
    rec, plane = prepare_device(u, v, w, vis, wt, spec, device=dev)
    if len(t) > 1 and np.any(np.diff(t.astype(np.int64)) < 0):
        # the exchange delivers (time_index, gindex) order: a stable sort by time
        order = torch.argsort(torch.from_numpy(t.astype(np.int64)).to(dev), stable=True)
        rec, plane = rec[order].contiguous(), plane[order].contiguous()
    g = spec.c_struct()
    counts = []
    off = 0
    for n_r in lens:   # messages of the exchange: per source partition and slab
        cnt = (C.c_int64 * R)()
        L.check(L.lib().wsb_route_count(ctx.handle, C.byref(g), S, R, None,
                                        _ptr(rec[off:off + n_r]) if n_r else None, n_r, cnt))
        counts.append([int(x) for x in cnt])
        off += n_r
    slabs = []
    if R > 1:
        from .distributed import CudaBackend
        srec, spl, per_slab = CudaBackend(dev).route(rec, plane, spec, S, R)
    else:
        srec, spl, per_slab = rec, plane, [rec.shape[0]]
    off = 0
    for d in range(R):
        sl = slab_of(spec, d, R)
        m = int(per_slab[d])
        out = ComplexGrid(spec, sl)
        if m:
            gp, _ = grid_slab_device(srec[off:off + m], spl[off:off + m], spec, kern, sl.v_start,
                                     sl.v_count)
            out.data[...] = unpack_grid_device(gp, spec, sl.v_start, sl.v_count).cpu().numpy()
        off += m
        slabs.append(out)
    log = log if log is not None else msglog.MessageLog()
    if R > 1:
        for msg in msglog.exchange_messages(topo, counts):
            log.append(msg)
        for msg in msglog.reduce_messages(topo, kind, spec.n_u, spec.n_v, spec.n_w):
            log.append(msg)
    return slabs, log


# ---------------------------------------------------------------------------
# dataset file (visdata.py:53-111, 262-341) and image files (transform.py:248-306)
# ---------------------------------------------------------------------------

_HEADER = struct.Struct("<4sIQIIIdd20s")


class FormatError(Exception):
    """Malformed dataset or image file (visdata.py:60-61)."""


def _record_dtype(n_chan: int) -> np.dtype:
    """visdata.py:262-272: 28 + 12 * n_chan bytes per record."""
    return np.dtype({"names": ["u", "v", "w", "time_index", "vis", "weight"],
                     "formats": ["<f8", "<f8", "<f8", "<u4", ("<f4", (n_chan, 2)),
                                 ("<f4", (n_chan,))],
                     "offsets": [0, 8, 16, 24, 28, 28 + 8 * n_chan],
                     "itemsize": 28 + 12 * n_chan})


@dataclass(frozen=True)
class ChunkSpec:
    """Which piece of a dataset to load (visdata.py:217-229): a frequency
    chunk keeps every record and a contiguous block of channels; a time chunk
    keeps every channel and the records of a contiguous block of time slices
    (partition_1d of the slices). The chunks of an axis cover the dataset
    exactly once."""
    axis: str
    chunk_index: int
    n_chunks: int

    def __post_init__(self):
        if self.axis not in ("frequency", "time"):
            raise ValueError(f"axis must be one of ('frequency', 'time'), got {self.axis!r}")
        if self.n_chunks < 1 or not (0 <= self.chunk_index < self.n_chunks):
            raise ValueError(f"chunk_index {self.chunk_index} outside range(0, {self.n_chunks})")


def read_dataset(path, chunk: ChunkSpec | None = None, rows: tuple | None = None):
    """Read an RVIS file (visdata.py:312-341): 64-byte header + records of
    28 + 12*n_chan bytes, optionally one ChunkSpec of it, or only the records
    [rows[0], rows[1]) (a rank's time partition). The file is memory mapped,
    so a chunk or row range reads only what it selects. Returns (header dict,
    dict of column arrays)."""
    path = Path(path)
    with open(path, "rb") as fh:
        head = fh.read(_HEADER.size)
    if len(head) < _HEADER.size:
        raise FormatError("truncated header")
    magic, version, n_rec, n_freq, n_corr, n_time, wmin, wmax, res = _HEADER.unpack(head)
    if magic != b"RVIS":
        raise FormatError(f"bad magic {magic!r}")
    if version != 1:
        raise FormatError(f"unsupported version {version}")
    n_chan = n_freq * n_corr
    rec_dt = _record_dtype(n_chan)
    body = path.stat().st_size - _HEADER.size
    if body != n_rec * rec_dt.itemsize:
        raise FormatError(f"truncated file: {body} payload bytes, expected {n_rec * rec_dt.itemsize}")
    packed = (np.memmap(path, dtype=rec_dt, mode="r", offset=_HEADER.size, shape=(n_rec,))
              if n_rec else np.zeros(0, dtype=rec_dt))
    if rows is not None:
        packed = packed[int(rows[0]):int(rows[1])]
    c0, c1 = 0, n_chan
    if chunk is not None and chunk.axis == "frequency":
        f0, fc = partition_1d(n_freq, chunk.n_chunks, chunk.chunk_index)   # visdata.py:297-300
        c0, c1 = f0 * n_corr, (f0 + fc) * n_corr
    elif chunk is not None:
        s0, sc = partition_1d(n_time, chunk.n_chunks, chunk.chunk_index)   # visdata.py:303-306
        t = np.asarray(packed["time_index"])
        packed = packed[(t >= s0) & (t < s0 + sc)]
    vis_ri = packed["vis"][:, c0:c1]
    vis = (vis_ri[..., 0] + 1j * vis_ri[..., 1]).astype(np.complex64)
    header = {"n_records": n_rec, "n_freq": n_freq, "n_corr": n_corr, "n_time_slices": n_time,
              "w_min_native": wmin, "w_max_native": wmax, "reserved": res}
    cols = {"u": np.ascontiguousarray(packed["u"]), "v": np.ascontiguousarray(packed["v"]),
            "w": np.ascontiguousarray(packed["w"]),
            "time_index": np.ascontiguousarray(packed["time_index"]),
            "vis": vis, "weight": np.ascontiguousarray(packed["weight"][:, c0:c1])}
    return header, cols


def write_dataset(cols: dict, header: dict, path) -> None:
    """Write an RVIS file (visdata.py:275-293 layout) from column arrays and
    a header dict as read_dataset returns them; read_dataset of the result is
    bit-identical."""
    n = len(cols["u"])
    n_chan = header["n_freq"] * header["n_corr"]
    if n != header["n_records"]:
        raise ValueError(f"header/record count mismatch: {header['n_records']} vs {n}")
    packed = np.zeros(n, dtype=_record_dtype(n_chan))
    for k in ("u", "v", "w", "time_index"):
        packed[k] = cols[k]
    vis = np.asarray(cols["vis"], np.complex64).reshape(n, n_chan)
    packed["vis"][..., 0] = vis.real
    packed["vis"][..., 1] = vis.imag
    packed["weight"] = np.asarray(cols["weight"], np.float32).reshape(n, n_chan)
    head = _HEADER.pack(b"RVIS", 1, n, header["n_freq"], header["n_corr"], header["n_time_slices"],
                        float(header["w_min_native"]), float(header["w_max_native"]),
                        bytes(header.get("reserved", b"")))
    with open(path, "wb") as fh:
        fh.write(head)
        fh.write(packed.tobytes())


def image_time_chunks(path, spec, kern, n_chunks: int, device: int = 0):
    """Dirty image of each time chunk of an RVIS dataset (ChunkSpec axis
    "time"), streamed: the next chunk is read and copied to the device while
    the current one is imaged (image_stream). Yields (FinalImage, diag)."""
    def batches():
        for i in range(n_chunks):
            _, c = read_dataset(path, ChunkSpec("time", i, n_chunks))
            yield c["u"], c["v"], c["w"], c["vis"], c["weight"]
    yield from image_stream(batches(), spec, kern, device=device)


def write_image(img: FinalImage, base_path, provenance: dict | None = None, pgm: bool = False):
    base = Path(base_path)
    base.parent.mkdir(parents=True, exist_ok=True)
    raw = base.with_suffix(".f64")
    raw.write_bytes(img.pixels.astype("<f8").tobytes())
    s = img.spec
    side = {"layout": "row-major (n_v, n_u) little-endian float64", "n_u": s.n_u, "n_v": s.n_v,
            "n_w": s.n_w, "cell_size_lm": s.cell_size_lm, "w_min_native": s.w_min_native,
            "w_max_native": s.w_max_native, "imag_residual_norm": img.imag_residual_norm,
            "real_norm": img.real_norm, "provenance": provenance or {}}
    js = base.with_suffix(".json")
    js.write_text(json.dumps(side, indent=2, sort_keys=True) + "\n")
    paths = {"raw": raw, "sidecar": js}
    if pgm:
        lo, hi = float(img.pixels.min()), float(img.pixels.max())
        scaled = (np.round((img.pixels - lo) / (hi - lo) * 255.0).astype(np.uint8) if hi > lo
                  else np.zeros(img.pixels.shape, np.uint8))
        p = base.with_suffix(".pgm")
        p.write_bytes(f"P5\n{img.pixels.shape[1]} {img.pixels.shape[0]}\n255\n".encode() + scaled.tobytes())
        paths["pgm"] = p
    return paths


# ---------------------------------------------------------------------------
# run_pipeline drop-in (pipeline.py:61-191)
# ---------------------------------------------------------------------------

def measure(meter, durations: dict, freq_level: str = "default") -> dict:
    """metrics.measure (metrics.py:183-193): per-phase joules from the meter's
    ``joules(durations, freq_level)``, plus their sum as "total" when the
    meter reports phases only."""
    for phase, seconds in durations.items():
        if seconds < 0:
            raise ValueError(f"negative duration for {phase}")
    joules = meter.joules(durations, freq_level)
    if "total" not in joules:
        joules = dict(joules)
        joules["total"] = sum(v for v in joules.values() if v is not None)
    return joules


def _partition_bounds(time_index: np.ndarray, n_ranks: int):
    """_partition_for_ranks (pipeline.py:47-58): the [lo, hi) record range of
    each rank -- contiguous groups of time slices (partition_time_ordered,
    visdata.py:344-366), or plain record runs when there are more ranks than
    slices. Also says whether the time-sorted check applies."""
    n = len(time_index)
    slices = np.unique(time_index)
    if n_ranks <= len(slices):
        out = []
        for r in range(n_ranks):
            s0, sc = partition_1d(len(slices), n_ranks, r)
            lo = int(np.searchsorted(time_index, slices[s0], side="left"))
            hi = int(np.searchsorted(time_index, slices[s0 + sc - 1], side="right"))
            out.append((lo, hi))
        return out, True
    return [(partition_1d(n, n_ranks, r)[0], sum(partition_1d(n, n_ranks, r)))
            for r in range(n_ranks)], False


def exchange_counts(cols, spec, half_support: int, bounds, device: int = 0):
    """Records each source rank's time partition sends to each v-slab of
    partition_1d(n_v, R) with the +-half_support halo predicate
    (comms.py:516-523), counted on the GPU (wsb_route_count). [R][R] ints."""
    R = len(bounds)
    rec, _plane = prepare_device(cols["u"], cols["v"], cols["w"], cols["vis"], cols["weight"],
                                 spec, device=device)
    ctx = context(rec.device)
    g = spec.c_struct()
    out = []
    for lo, hi in bounds:
        cnt = (C.c_int64 * R)()
        sub = rec[lo:hi]
        L.check(L.lib().wsb_route_count(ctx.handle, C.byref(g), int(half_support), R, None,
                                        _ptr(sub) if hi > lo else None, hi - lo, cnt))
        out.append([int(x) for x in cnt])
    return out


def run_pipeline(dataset_path, n_u: int, n_v: int, n_w: int, cell_size_lm: float, kernel,
                 topo=None, strategy=None, meter=None, freq_level: str = "default",
                 label: str = "run", out_dir=None, pgm: bool = False, seed=None,
                 device: int = 0) -> PipelineResult:
    """Same call, result type and error behaviour as the reference
    run_pipeline (pipeline.py:61-191); the gridding, FFT and w-stacking
    phases run on the B200 through wsb_image.

    ``topo`` (a reference Topology, default 1x1) and ``strategy`` (default
    ReduceStrategy("direct", True)) keep their meaning for everything the
    caller can observe: the records are split into the ranks' time
    partitions (pipeline.py:47-58; unsorted time_index raises ValueError as
    partition_time_ordered does), and the returned MessageLog, messages.csv
    and ``ops`` byte / message totals are those of the reference's virtual
    choreography on ``topo`` (msglog.py; exchange counts measured on the
    GPU). The image itself does not depend on the topology (the reference
    guarantees bit-identical grids for any rank count, gridder.py:267-268)
    and is computed once on ``device``. Multi-GPU imaging of a dataset is
    ``distributed.run_pipeline_distributed`` (one process per GPU, each
    reading its own time partition).
    ``meter``: any object with ``start()`` and ``joules(durations,
    freq_level)`` (the reference's meters, energy.NvmlRaplMeter); per-phase
    joules as metrics.measure returns them (pipeline.py:173-176)."""
    from . import msglog
    kern = as_kernel_spec(kernel)
    kind = getattr(strategy, "kind", "direct") if strategy is not None else "direct"
    if kind not in msglog.REDUCE_KINDS:
        raise ValueError(f"reduce kind must be one of {msglog.REDUCE_KINDS}, got {kind!r}")
    R = int(topo.n_ranks) if topo is not None else 1
    if meter is not None and hasattr(meter, "start"):
        meter.start()
    t_begin = time.perf_counter()
    times = {}
    t0 = time.perf_counter()
    header, cols = read_dataset(dataset_path)
    spec = GridSpec(n_u=n_u, n_v=n_v, n_w=n_w, cell_size_lm=cell_size_lm,
                    w_min_native=header["w_min_native"], w_max_native=header["w_max_native"])
    t_idx = cols["time_index"]
    bounds, time_ordered = _partition_bounds(t_idx, R)
    times["read"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    img, diag = image(cols["u"], cols["v"], cols["w"], t_idx if time_ordered else None,
                      cols["vis"], cols["weight"], spec, kern, device=device)
    wall = time.perf_counter() - t0
    pm = diag["phase_ms"]
    # exclusive segments of the device timeline, scaled into the call's wall time
    dev_total = max(pm[6], 1e-9)
    scale = min(1.0, wall / (dev_total / 1e3))
    times["read"] += pm[0] / 1e3 * scale          # host -> device copies
    times["gridding"] = pm[1] / 1e3 * scale
    times["reduce"] = 0.0                         # the identity after the exchange
    times["fft"] = pm[3] / 1e3 * scale
    times["wcorrect"] = pm[4] / 1e3 * scale
    t0 = time.perf_counter()
    if R > 1:
        counts = exchange_counts(cols, spec, kern.half_support, bounds, device=device)
        log = msglog.virtual_log(topo, kind, n_u, n_v, n_w, counts)
    else:
        log = msglog.MessageLog()
    paths = {}
    if out_dir is not None:
        out_dir = Path(out_dir)
        out_dir.mkdir(parents=True, exist_ok=True)
        prov = {"dataset": str(dataset_path),
                "kernel": {"kind": kern.kind, "half_support": kern.half_support,
                           "shape_param": kern.shape_param},
                "topology": ({"n_nodes": topo.n_nodes, "ranks_per_node": topo.ranks_per_node,
                              "threads_per_rank": topo.threads_per_rank}
                             if topo is not None else None),
                "strategy": {"kind": kind,
                             "deterministic": getattr(strategy, "deterministic", True)},
                "engine": "wsb-b200", "seed": seed}
        paths = write_image(img, out_dir / "image", prov, pgm=pgm)
        log.to_csv(out_dir / "messages.csv")
        paths["messages"] = out_dir / "messages.csv"
    times["write"] = time.perf_counter() - t0 + pm[5] / 1e3 * scale
    times["total"] = time.perf_counter() - t_begin
    energy = {}
    if meter is not None:
        energy = measure(meter, {k: v for k, v in times.items() if k != "total"}, freq_level)
    ops = {"records": len(cols["u"]), "grid_updates": diag["grid_updates"],
           "exchange_bytes": log.total_bytes(phase="exchange"),
           "reduce_bytes": log.total_bytes(phase="reduce"),
           "fft_bytes": log.total_bytes(phase="fft"),
           "reduce_messages": log.count(phase="reduce"), "stack_pixels": n_u * n_v}
    run = RunRecord(label=label, topology=topo, freq_level=freq_level, phase_times=times,
                    energy_joules=energy)
    return PipelineResult(run=run, image=img, log=log, ops=ops, paths=paths)
