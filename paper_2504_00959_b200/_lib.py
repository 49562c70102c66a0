"""ctypes binding of libwsb.so (include/wsb.h).

The library is the only compute path: there is no CPU fallback. Loading
fails loudly when the shared object is missing; calls fail loudly when no
CUDA device is present.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("WSB_LIB", Path(__file__).resolve().parent / "libwsb.so"))

WSB_OK = 0
WSB_EINVAL = -1
WSB_ECUDA = -2
WSB_ENCCL = -3
WSB_ENOMEM = -4
WSB_EUNSUPPORTED = -5
P_GROUP = 1
STRIP = 16          # WSB_STRIP: column width of the gridder's strip layout
ITEM_COLS = 16      # WSB_ITEM_COLS: columns of one gridder work item (K1 keys)
EXEC_ENERGY = 1
KERNEL_GAUSSIAN = 0
KERNEL_KAISER_BESSEL = 1

# every symbol include/wsb.h declares
EXPORTS = (
    "wsb_strerror", "wsb_last_error", "wsb_version", "wsb_ctx_create", "wsb_ctx_destroy",
    "wsb_ctx_set_stream", "wsb_ctx_trim", "wsb_image", "wsb_image_device", "wsb_prepare",
    "wsb_route_count", "wsb_route_pack", "wsb_grid_slab", "wsb_fft_rows", "wsb_fft_cols_stack",
    "wsb_grid_unpack", "wsb_tiles_debug", "wsb_last_timings", "wsb_row_histogram",
    "wsb_fft_rows_peer", "wsb_push_blocks", "wsb_ctx_set_precision", "wsb_route_planes_count",
    "wsb_route_planes_pack", "wsb_fft_cols_partial", "wsb_image_finish", "wsb_plane_histogram",
    "wsb_grid_unpack_rows", "wsb_ctx_set_energy", "wsb_bucket_items",
)


class WsbGrid(C.Structure):
    _fields_ = [("n_u", C.c_int32), ("n_v", C.c_int32), ("n_w", C.c_int32), ("reserved", C.c_int32),
                ("cell_size_lm", C.c_double), ("w_min_native", C.c_double),
                ("w_max_native", C.c_double)]


class WsbKernel(C.Structure):
    _fields_ = [("kind", C.c_int32), ("half_support", C.c_int32), ("shape_param", C.c_double)]


class WsbExec(C.Structure):
    _fields_ = [("device", C.c_int32), ("precision", C.c_int32), ("deterministic", C.c_int32),
                ("flags", C.c_int32)]


class WsbDiag(C.Structure):
    _fields_ = [("imag_residual_norm", C.c_double), ("real_norm", C.c_double),
                ("grid_updates", C.c_int64), ("records", C.c_int64), ("tile_entries", C.c_int64),
                ("phase_ms", C.c_double * 7), ("exchanged_records", C.c_int64),
                ("gpu_joules", C.c_double), ("host_joules", C.c_double)]


class WsbError(RuntimeError):
    pass


_lib = None


def lib() -> C.CDLL:
    """Load libwsb.so, building it first when it is missing (unless
    WSB_NO_AUTOBUILD is set). A library older than its sources is loaded as
    is, with a warning: rebuild with ``python -m paper_2504_00959_b200.build``
    (the driver's build() step does). Raises if the library cannot be loaded."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists() and os.environ.get("WSB_NO_AUTOBUILD") is None:
        from .build import build
        build()
    if LIB_PATH.exists() and LIB_PATH == Path(__file__).resolve().parent / "libwsb.so":
        from .build import stale_sources
        newer = stale_sources(LIB_PATH)
        if newer:
            import warnings
            warnings.warn(f"{LIB_PATH.name} is older than {', '.join(newer[:3])}: "
                          "rebuild with python -m paper_2504_00959_b200.build", stacklevel=2)
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: run python -m paper_2504_00959_b200.build")
    L = C.CDLL(str(LIB_PATH))
    p, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    G, K, E, D = C.POINTER(WsbGrid), C.POINTER(WsbKernel), C.POINTER(WsbExec), C.POINTER(WsbDiag)
    sig = {
        "wsb_strerror": (C.c_char_p, [C.c_int]),
        "wsb_last_error": (C.c_char_p, []),
        "wsb_version": (C.c_int, []),
        "wsb_ctx_create": (C.c_int, [i32, C.POINTER(p)]),
        "wsb_ctx_destroy": (C.c_int, [p]),
        "wsb_ctx_set_stream": (C.c_int, [p, p]),
        "wsb_ctx_trim": (C.c_int, [p]),
        "wsb_image": (C.c_int, [G, K, E, p, p, p, p, p, p, i64, i32, p, D]),
        "wsb_image_device": (C.c_int, [p, G, K, p, p, p, p, p, i64, i32, p, D]),
        "wsb_prepare": (C.c_int, [p, G, p, p, p, p, p, i64, i32, p, p]),
        "wsb_route_count": (C.c_int, [p, G, i32, i32, p, p, i64, p]),
        "wsb_route_pack": (C.c_int, [p, G, i32, i32, p, p, p, i64, p, p, p]),
        "wsb_row_histogram": (C.c_int, [p, G, p, i64, p]),
        "wsb_plane_histogram": (C.c_int, [p, G, p, i64, p]),
        "wsb_route_planes_count": (C.c_int, [p, G, i32, p, p, p, i64, p]),
        "wsb_route_planes_pack": (C.c_int, [p, G, i32, p, p, p, i64, p, p, p]),
        "wsb_fft_cols_partial": (C.c_int, [p, G, i32, i32, i32, i32, p, p]),
        "wsb_image_finish": (C.c_int, [p, G, p, p, p]),
        "wsb_grid_slab": (C.c_int, [p, G, K, i32, i32, p, p, i64, p, p]),
        "wsb_fft_rows": (C.c_int, [p, G, i32, p, p, i32, i32, i32, p]),
        "wsb_fft_rows_peer": (C.c_int, [p, G, i32, p, i32, i32, i32, p, p]),
        "wsb_push_blocks": (C.c_int, [p, i32, p, p, p]),
        "wsb_ctx_set_precision": (C.c_int, [p, i32]),
        "wsb_ctx_set_energy": (C.c_int, [p, i32]),
        "wsb_fft_cols_stack": (C.c_int, [p, G, i32, p, i32, i32, i32, i32, p, p, p]),
        "wsb_grid_unpack": (C.c_int, [p, G, i32, i32, p, p]),
        "wsb_grid_unpack_rows": (C.c_int, [p, G, i32, i32, i32, i32, p, p]),
        "wsb_tiles_debug": (C.c_int, [p, p, p, p, p]),
        "wsb_bucket_items": (C.c_int, [p, G, i32, i32, i32, p, p, i64, p, p, p, p, p, p]),
        "wsb_last_timings": (C.c_int, [p, p, p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a WSB_E* code to the reference's exception types
    (ValueError for invalid specs/inputs, mesh.py:79-95, visdata.py:178-184)."""
    if rc == WSB_OK:
        return
    L = lib()
    msg = f"{L.wsb_strerror(rc).decode()}: {L.wsb_last_error().decode()}"
    if rc == WSB_EINVAL:
        raise ValueError(msg)
    if rc == WSB_ENOMEM:
        raise MemoryError(msg)
    if rc == WSB_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise WsbError(msg)


def grid_struct(n_u, n_v, n_w, cell, w_min_native, w_max_native) -> WsbGrid:
    return WsbGrid(int(n_u), int(n_v), int(n_w), 0, float(cell), float(w_min_native),
                   float(w_max_native))


def kernel_struct(kind: int, half_support: int, shape: float) -> WsbKernel:
    return WsbKernel(int(kind), int(half_support), float(shape))


class Context:
    """One libwsb context per CUDA device, bound to torch's current stream."""

    _per_device: dict = {}

    def __init__(self, device: int):
        self.device = device
        h = C.c_void_p()
        check(lib().wsb_ctx_create(int(device), C.byref(h)))
        self.handle = h

    @classmethod
    def get(cls, device: int) -> "Context":
        c = cls._per_device.get(device)
        if c is None:
            c = cls._per_device[device] = cls(device)
        return c

    def bind_stream(self, stream_ptr: int) -> None:
        check(lib().wsb_ctx_set_stream(self.handle, C.c_void_p(stream_ptr)))
