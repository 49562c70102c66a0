"""CPU-side checks of the C ABI library: it loads, exports every symbol
include/wsb.h declares, and reports errors without touching a GPU."""

import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def L():
    from paper_2504_00959_b200 import _lib
    return _lib


def test_header_and_binding_agree(L):
    hdr = (ROOT / "include" / "wsb.h").read_text()
    declared = set(re.findall(r"\b(wsb_[a-z_]+)\s*\(", hdr))
    assert declared == set(L.EXPORTS)


def test_library_exports_every_symbol(L):
    lib = L.lib()
    for name in L.EXPORTS:
        assert hasattr(lib, name), name


def test_version_and_strerror(L):
    lib = L.lib()
    assert lib.wsb_version() == 100
    assert lib.wsb_strerror(-1) == b"invalid argument"
    assert lib.wsb_strerror(0) == b"ok"


def test_struct_sizes_match_header(L):
    assert C.sizeof(L.WsbGrid) == 40
    assert C.sizeof(L.WsbKernel) == 16
    assert C.sizeof(L.WsbExec) == 16
    assert C.sizeof(L.WsbDiag) == 2 * 8 + 3 * 8 + 7 * 8 + 8 + 2 * 8


def test_invalid_grid_rejected_before_any_launch(L):
    lib = L.lib()
    g = L.grid_struct(48, 64, 4, 1e-3, 0.0, 0.0)        # n_u not a power of two
    k = L.kernel_struct(0, 3, 1.0)
    out = (C.c_double * 4)()
    rc = lib.wsb_image(C.byref(g), C.byref(k), None, None, None, None, None, None, None, 0, 1,
                       out, None)
    assert rc == L.WSB_EINVAL
    assert b"power of two" in lib.wsb_last_error()
    with pytest.raises(ValueError):
        L.check(rc)


def test_invalid_kernel_rejected(L):
    lib = L.lib()
    g = L.grid_struct(64, 64, 4, 1e-3, 0.0, 0.0)
    k = L.kernel_struct(0, 0, 1.0)
    out = (C.c_double * 4)()
    assert lib.wsb_image(C.byref(g), C.byref(k), None, None, None, None, None, None, None, 0, 1,
                         out, None) == L.WSB_EINVAL


def test_host_specs_validate_like_reference():
    import paper_2504_00959_b200 as W
    with pytest.raises(ValueError):
        W.GridSpec(4096, 4096, 4, 1e-3)
    with pytest.raises(ValueError):
        W.KernelSpec("boxcar", 1, 1.0)
    assert W.KernelSpec.kaiser_bessel(5).shape_param == pytest.approx(11.7)
    assert W.partition_1d(4096, 16, 3) == (768, 256)


def test_product_never_imports_oracle():
    for p in (ROOT / "paper_2504_00959_b200").rglob("*.py"):
        src = p.read_text()
        assert "from oracle" not in src and "import oracle" not in src, p
