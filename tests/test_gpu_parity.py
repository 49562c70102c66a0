"""GPU parity: libwsb.so (through the C ABI) against the pinned oracle and the
reference-generated golden fixtures. Needs a B200."""

import numpy as np
import pytest

from conftest import chunk_from, rel_l2
from oracle import wstack_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_00959_b200 as W
    return W


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


@pytest.mark.parametrize("name", ["syn", "edge"])
def test_prepare_bitexact(W, golden_bucket, name):
    g = golden_bucket
    n_u, n_v, n_w, S = (int(x) for x in g[f"{name}_spec"])
    u, v, w, t, vis, wt = chunk_from(g, f"{name}_in_")
    spec = W.GridSpec(n_u, n_v, n_w, 1e-3)
    rec, plane = W.prepare_device(u, v, w, vis, wt, spec)
    rec = rec.cpu().numpy()
    assert np.array_equal(_bits(rec[:, 0]), _bits(g[f"{name}_prep_gu"]))
    assert np.array_equal(_bits(rec[:, 1]), _bits(g[f"{name}_prep_gv"]))
    assert np.array_equal(plane.cpu().numpy().astype(np.uint32), g[f"{name}_prep_plane"])
    val = g[f"{name}_prep_value"]
    assert np.array_equal(_bits(rec[:, 2]), _bits(val.real.copy()))
    assert np.array_equal(_bits(rec[:, 3]), _bits(val.imag.copy()))


@pytest.mark.parametrize("name", ["syn", "edge"])
@pytest.mark.parametrize("R", [2, 4, 8])
def test_route_bitexact(W, golden_bucket, name, R):
    """Destination slabs (comms.py:516-523) and arrival order vs the
    reference's SectorBatch columns."""
    import ctypes as C
    from paper_2504_00959_b200 import _lib as L
    from paper_2504_00959_b200.imager import context, _ptr
    g = golden_bucket
    n_u, n_v, n_w, S = (int(x) for x in g[f"{name}_spec"])
    u, v, w, t, vis, wt = chunk_from(g, f"{name}_in_")
    spec = W.GridSpec(n_u, n_v, n_w, 1e-3)
    rec, plane = W.prepare_device(u, v, w, vis, wt, spec)
    ctx = context(rec.device)
    counts = (C.c_int64 * R)()
    gs = spec.c_struct()
    L.check(L.lib().wsb_route_count(ctx.handle, C.byref(gs), S, R, None, _ptr(rec), rec.shape[0],
                                    counts))
    tot = sum(counts)
    srec = torch.empty((tot, 4), dtype=torch.float64, device=rec.device)
    spl = torch.empty(tot, dtype=torch.int32, device=rec.device)
    sidx = torch.empty(tot, dtype=torch.int64, device=rec.device)
    L.check(L.lib().wsb_route_pack(ctx.handle, C.byref(gs), S, R, None, _ptr(rec), _ptr(plane),
                                   rec.shape[0], _ptr(srec), _ptr(spl), _ptr(sidx)))
    srec, spl, sidx = srec.cpu().numpy(), spl.cpu().numpy(), sidx.cpu().numpy()
    off = 0
    for d in range(R):
        key = f"{name}_R{R}_d{d}_"
        n_d = int(counts[d])
        assert n_d == len(g[key + "gu"])
        sl = slice(off, off + n_d)
        assert np.array_equal(sidx[sl].astype(np.uint64), g[key + "gindex"])
        assert np.array_equal(_bits(srec[sl, 0]), _bits(g[key + "gu"]))
        assert np.array_equal(_bits(srec[sl, 1]), _bits(g[key + "gv"]))
        assert np.array_equal(spl[sl].astype(np.uint32), g[key + "plane"])
        assert np.array_equal(_bits(srec[sl, 2]), _bits(g[key + "value"].real.copy()))
        off += n_d


@pytest.mark.parametrize("kname", ["gauss3", "gauss1", "kb1", "kb3", "kb5"])
def test_grid_matches_reference(W, golden_grid, kname):
    g = golden_grid
    S = int(g[f"{kname}_S"][0])
    shape = float(g[f"{kname}_shape"][0])
    kind = "gaussian" if kname.startswith("gauss") else "kaiser_bessel"
    spec = W.GridSpec(64, 64, 4, 1e-3, w_max_native=12.0)
    kern = W.KernelSpec(kind, S, shape)
    u, v, w, t, vis, wt = chunk_from(g, "in_")
    rec, plane = W.prepare_device(u, v, w, vis, wt, spec)
    gp, upd = W.grid_slab_device(rec, plane, spec, kern, 0, 64)
    grid = W.unpack_grid_device(gp, spec, 0, 64).cpu().numpy()
    assert upd == int(g[f"{kname}_updates"][0])
    assert np.max(np.abs(grid - g[f"{kname}_grid"])) <= 1e-12


@pytest.mark.parametrize("S,beta", [(1, 12.0), (3, 30.0), (2, 4.68)])
def test_grid_kaiser_bessel_any_beta(W, golden_grid, S, beta):
    """Kaiser-Bessel weights: the power-series evaluation (default betas) and
    the np.i0 Chebyshev fallback (betas beyond the series length) both match
    the oracle's np.i0 kernel (gridder.py:92-98) to 1e-12."""
    g = golden_grid
    spec = W.GridSpec(64, 64, 4, 1e-3, w_max_native=12.0)
    kern = W.KernelSpec("kaiser_bessel", S, beta)
    u, v, w, t, vis, wt = chunk_from(g, "in_")
    rec, plane = W.prepare_device(u, v, w, vis, wt, spec)
    gp, upd = W.grid_slab_device(rec, plane, spec, kern, 0, 64)
    grid = W.unpack_grid_device(gp, spec, 0, 64).cpu().numpy()
    prep = O.prepare(u, v, w, t, vis, wt, 64, 64, 4)
    batch = O.exchange([prep], 64, 1, S)[0]
    ref, upd_ref = O.grid_slab(batch, 64, 4, O.KIND_KAISER_BESSEL, S, beta, 0, 64)
    assert upd == upd_ref
    assert np.max(np.abs(grid - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("kind,S", [("gaussian", 2), ("gaussian", 4), ("gaussian", 5),
                                    ("gaussian", 6), ("gaussian", 7), ("kaiser_bessel", 4),
                                    ("kaiser_bessel", 7)])
def test_grid_every_support_vs_oracle(W, kind, S):
    """Every K2 instantiation (half supports 1..7: two- and three-tile
    windows) against the oracle's grid_slab, on dense random records that
    fill single items beyond one work part (split items) and reach the mesh
    edges; grid_updates equal."""
    rng = np.random.default_rng(100 + S)
    n = 40000
    u = np.concatenate([rng.random(n // 2), 0.30 + 0.02 * rng.random(n // 2)])   # a dense patch
    v = np.concatenate([rng.random(n // 2), 0.60 + 0.02 * rng.random(n // 2)])
    w = rng.random(n)
    t = np.zeros(n, np.uint32)
    vis = (rng.standard_normal((n, 1)) + 1j * rng.standard_normal((n, 1))).astype(np.complex64)
    wt = rng.uniform(0.5, 1.5, (n, 1)).astype(np.float32)
    spec = W.GridSpec(128, 128, 3, 1e-3, w_max_native=10.0)
    shape = 1.0 if kind == "gaussian" else 2.34 * S
    kern = W.KernelSpec(kind, S, shape)
    rec, plane = W.prepare_device(u, v, w, vis, wt, spec)
    gp, upd = W.grid_slab_device(rec, plane, spec, kern, 0, 128)
    grid = W.unpack_grid_device(gp, spec, 0, 128).cpu().numpy()
    prep = O.prepare(u, v, w, t, vis, wt, 128, 128, 3)
    batch = O.exchange([prep], 128, 1, S)[0]
    ref, upd_ref = O.grid_slab(batch, 128, 3, O.KIND_GAUSSIAN if kind == "gaussian" else O.KIND_KAISER_BESSEL,
                               S, shape, 0, 128)
    assert upd == upd_ref
    assert np.max(np.abs(grid - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_grid_records_at_item_corners_four_entries_each(W):
    """Every record's footprint straddles two 16-column strips and two
    128-row blocks: four K1 entries per record, above the entry buffers'
    first sizing (2 per record), so K1 re-runs with exact buffers; the grid
    still equals the oracle's and grid_updates the reference count."""
    rng = np.random.default_rng(11)
    n = 30000
    n_u, n_v = 64, 256
    ci = rng.integers(1, n_u // 16, n) * 16          # strip boundaries 16, 32, 48
    u = (ci + rng.uniform(-2.0, 2.0, n)) / n_u
    v = (128 + rng.uniform(-2.0, 2.0, n)) / n_v       # the row-block boundary 128
    w = rng.random(n)
    t = np.zeros(n, np.uint32)
    vis = (rng.standard_normal((n, 1)) + 1j * rng.standard_normal((n, 1))).astype(np.complex64)
    wt = np.ones((n, 1), np.float32)
    spec = W.GridSpec(n_u, n_v, 2, 1e-3, w_max_native=10.0)
    kern = W.KernelSpec.gaussian(3, 1.0)
    from paper_2504_00959_b200 import _lib as L
    dev = torch.cuda.current_device()
    saved = L.Context._per_device.get(dev)
    L.Context._per_device[dev] = L.Context(dev)        # fresh buffers: the first sizing applies
    try:
        rec, plane = W.prepare_device(u, v, w, vis, wt, spec)
        keys, idx, off, ib = W.bucket_items_device(rec, plane, spec, 3, 0, n_v)
        assert len(keys) > 3.5 * n                     # ~4 entries per record
        gp, upd = W.grid_slab_device(rec, plane, spec, kern, 0, n_v)
        grid = W.unpack_grid_device(gp, spec, 0, n_v).cpu().numpy()
    finally:
        L.Context._per_device[dev] = saved
    prep = O.prepare(u, v, w, t, vis, wt, n_u, n_v, 2)
    batch = O.exchange([prep], n_v, 1, 3)[0]
    ref, upd_ref = O.grid_slab(batch, n_u, 2, O.KIND_GAUSSIAN, 3, 1.0, 0, n_v)
    assert upd == upd_ref
    assert np.max(np.abs(grid - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("R", [2, 4])
def test_grid_slabs_bitwise_across_slab_counts(W, golden_grid, R):
    """Per-slab gridding after the exchange reproduces the 1-slab grid
    bit for bit (gridder.py:267-268)."""
    g = golden_grid
    spec = W.GridSpec(64, 64, 4, 1e-3, w_max_native=12.0)
    kern = W.KernelSpec("gaussian", 3, 1.0)
    u, v, w, t, vis, wt = chunk_from(g, "in_")
    rec, plane = W.prepare_device(u, v, w, vis, wt, spec)
    full, upd_full = W.grid_slab_device(rec, plane, spec, kern, 0, 64)
    full = W.unpack_grid_device(full, spec, 0, 64).cpu().numpy()
    parts, upd_sum = [], 0
    gv = rec[:, 1].cpu().numpy()
    for d in range(R):
        v0, vc = W.partition_1d(64, R, d)
        m = (gv + 3 >= v0) & (gv - 3 <= v0 + vc - 1)
        idx = torch.from_numpy(np.nonzero(m)[0]).to(rec.device)
        gp, upd = W.grid_slab_device(rec[idx].contiguous(), plane[idx].contiguous(), spec, kern, v0, vc)
        parts.append(W.unpack_grid_device(gp, spec, v0, vc).cpu().numpy())
        upd_sum += upd
    assert upd_sum == upd_full
    assert np.concatenate(parts, axis=1).tobytes() == full.tobytes()


@pytest.mark.parametrize("name", ["small", "kb5", "kb1", "nw1", "wide", "multichan"])
def test_image_matches_reference(W, golden_image, name):
    g = golden_image
    n_u, n_v, n_w, S, _ = (int(x) for x in g[f"{name}_cfg"])
    cell, wmin, wmax, shape = (float(x) for x in g[f"{name}_fcfg"])
    kind = "gaussian" if int(g[f"{name}_kind"][0]) == 0 else "kaiser_bessel"
    spec = W.GridSpec(n_u, n_v, n_w, cell, w_min_native=wmin, w_max_native=wmax)
    kern = W.KernelSpec(kind, S, shape)
    img, diag = W.image(*chunk_from(g, f"{name}_in_"), spec, kern)
    assert diag["grid_updates"] == int(g[f"{name}_grid_updates"][0])
    err = rel_l2(img.pixels, g[f"{name}_pixels"])
    assert err <= 1e-10, err
    np.testing.assert_allclose([img.imag_residual_norm, img.real_norm], g[f"{name}_norms"],
                               rtol=1e-9, atol=1e-300)


def test_image_medium_vs_oracle(W):
    """256x256x8, 200k records, KB S=3, w up to 400: GPU vs oracle."""
    src = ((0.02, -0.015, 2.0), (0.0, 0.0, 1.0), (-0.03, 0.01, 0.5))
    u, v, w, t, vis, wt = O.generate_synthetic(src, 200_000, 1, seed=21, cell_size_lm=5e-4,
                                               w_max_native=400.0)
    spec = W.GridSpec(256, 256, 8, 5e-4, w_max_native=400.0)
    kern = W.KernelSpec.kaiser_bessel(3)
    ref = O.image(u, v, w, t, vis, wt, 256, 256, 8, 5e-4, 0.0, 400.0, O.KIND_KAISER_BESSEL, 3,
                  kern.shape_param)
    img, diag = W.image(u, v, w, t, vis, wt, spec, kern)
    assert diag["grid_updates"] == ref["grid_updates"]
    assert rel_l2(img.pixels, ref["pixels"]) <= 1e-10


def test_image_deterministic_and_device_path(W, golden_image):
    g = golden_image
    n_u, n_v, n_w, S, _ = (int(x) for x in g["wide_cfg"])
    cell, wmin, wmax, shape = (float(x) for x in g["wide_fcfg"])
    spec = W.GridSpec(n_u, n_v, n_w, cell, w_min_native=wmin, w_max_native=wmax)
    kern = W.KernelSpec("gaussian", S, shape)
    u, v, w, t, vis, wt = chunk_from(g, "wide_in_")
    a, _ = W.image(u, v, w, t, vis, wt, spec, kern)
    b, _ = W.image(u, v, w, t, vis, wt, spec, kern)
    dev = torch.device("cuda", 0)
    c, _ = W.image_device(torch.from_numpy(u).to(dev), torch.from_numpy(v).to(dev),
                          torch.from_numpy(w).to(dev), torch.from_numpy(vis).to(dev),
                          torch.from_numpy(wt).to(dev), spec, kern)
    assert a.pixels.tobytes() == b.pixels.tobytes()
    assert a.pixels.tobytes() == c.cpu().numpy().tobytes()


def test_invalid_inputs_raise_value_error(W):
    spec = W.GridSpec(32, 32, 2, 1e-3)
    kern = W.KernelSpec()
    one = np.ones((1, 1), np.complex64)
    with pytest.raises(ValueError):
        W.image([1.0], [0.5], [0.5], None, one, np.ones((1, 1), np.float32), spec, kern)
    with pytest.raises(ValueError):
        W.image([0.5], [0.5], [1.5], None, one, np.ones((1, 1), np.float32), spec, kern)
    with pytest.raises(ValueError):
        W.image([0.5], [0.5], [0.5], None, one, -np.ones((1, 1), np.float32), spec, kern)
    with pytest.raises(ValueError):
        W.image([np.nan], [0.5], [0.5], None, one, np.ones((1, 1), np.float32), spec, kern)


def test_empty_input_gives_zero_image(W):
    spec = W.GridSpec(32, 32, 2, 1e-3)
    img, diag = W.image(np.zeros(0), np.zeros(0), np.zeros(0), None, np.zeros((0, 1), np.complex64),
                        np.zeros((0, 1), np.float32), spec, W.KernelSpec())
    assert diag["grid_updates"] == 0
    assert not np.any(img.pixels)


@pytest.mark.gpu
def test_route_uneven_slabs_and_row_histogram(W, golden_bucket):
    """Explicit (load-balanced) slab starts: the packed records of each slab
    are exactly the oracle's halo selection (comms.py:521-523) in gindex
    order; the row histogram is the bincount of floor(gv)."""
    import ctypes as C
    from oracle import wstack_oracle as O
    from paper_2504_00959_b200 import _lib as L
    from paper_2504_00959_b200.distributed import CudaBackend
    g = golden_bucket
    n_u, n_v, n_w, S = (int(x) for x in g["syn_spec"])
    u, v, w, t, vis, wt = chunk_from(g, "syn_in_")
    spec = W.GridSpec(n_u, n_v, n_w, 1e-3)
    be = CudaBackend(0)
    rec, plane = be.prepare(u, v, w, vis, wt, spec)
    gv = rec[:, 1].cpu().numpy()
    hist = be.row_histogram(rec, spec).cpu().numpy()
    assert np.array_equal(hist, np.bincount(np.floor(gv).astype(np.int64), minlength=n_v))
    R = 3
    starts = [0, n_v // 5, n_v // 5 + 3, n_v]
    srec, spl, counts = be.route(rec, plane, spec, S, R, starts)
    srec = srec.cpu().numpy()
    off = 0
    for d in range(R):
        m = O.halo_mask(gv, S, starts[d], starts[d + 1] - starts[d])
        assert counts[d] == int(m.sum())
        assert _bits(srec[off:off + counts[d], 1]).tobytes() == _bits(gv[m]).tobytes()
        off += counts[d]
    # invalid starts are rejected
    gs = spec.c_struct()
    bad = (C.c_int32 * 4)(0, 10, 10, n_v)
    cnt = (C.c_int64 * 3)()
    with pytest.raises(ValueError):
        L.check(L.lib().wsb_route_count(be.ctx.handle, C.byref(gs), S, 3, bad,
                                        C.c_void_p(rec.data_ptr()), rec.shape[0], cnt))


@pytest.mark.parametrize("n", [8192, 16384])
def test_large_mesh_split_transforms(W, n):
    """Rows/columns longer than the on-chip 4096 points (cfg4's 16384²) run
    as SP = n/4096 decimation-in-frequency residue transforms. The image is
    checked against the reference formulas (transform.py:173-230: sign,
    normalised inverse 2D DFT, w screen skipped at w_k = 0, stack / n_w * n)
    evaluated with torch's FP64 FFT on the GPU grid itself, to 1e-10."""
    import torch
    rng = np.random.default_rng(5)
    m = 20_000
    n_w = 2
    cell = 2e-5
    spec = W.GridSpec(n, n, n_w, cell, w_max_native=800.0)
    kern = W.KernelSpec.gaussian(3, 1.0)
    u = rng.uniform(0.3, 0.7, m)
    v = rng.uniform(0.3, 0.7, m)
    w = rng.uniform(0.0, 1.0, m)
    vis = (rng.standard_normal(m) + 1j * rng.standard_normal(m)).astype(np.complex64)
    wt = rng.uniform(0.5, 1.0, m).astype(np.float32)
    dev = torch.device("cuda", 0)
    du, dv, dw, dvis, dwt = (torch.from_numpy(a).to(dev) for a in (u, v, w, vis, wt))
    img, diag = W.image_device(du, dv, dw, dvis, dwt, spec, kern)
    rec, plane = W.prepare_device(du, dv, dw, dvis, dwt, spec)
    gs, upd = W.grid_slab_device(rec, plane, spec, kern, 0, n)
    assert upd == diag["grid_updates"]
    grid = W.unpack_grid_device(gs, spec, 0, n)          # (n_w, n_v, n_u), no sign
    del gs
    ii = torch.arange(n, device=dev, dtype=torch.float64)
    sign = 1.0 - 2.0 * ((ii[:, None] + ii[None, :]).remainder(2.0))
    l = (ii - n // 2) * cell
    nn = torch.sqrt(1.0 - l[None, :] ** 2 - l[:, None] ** 2)
    acc = torch.zeros((n, n), dtype=torch.complex128, device=dev)
    for k in range(n_w):
        p = torch.fft.ifft2(grid[k] * sign)
        wk = spec.plane_w_native(k)
        if wk != 0.0:
            p = p * torch.exp(2j * np.pi * wk * (nn - 1.0))
        acc = acc + p
        del p
    acc = acc / n_w * nn
    ref = acc.real
    got = img if isinstance(img, torch.Tensor) else torch.as_tensor(img.pixels, device=dev)
    err = float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))
    assert err <= 1e-10, err
    assert abs(diag["imag_residual_norm"] - float(torch.linalg.norm(acc.imag))) <= 1e-9 * float(
        torch.linalg.norm(acc.imag))


def test_image_stream_matches_single_calls(W, golden_image):
    """The double-buffered stream API returns, batch by batch, exactly the
    images of separate wsb_image calls (the copies overlap, the math does
    not change)."""
    import torch
    g = golden_image
    n_u, n_v, n_w, S, _ = (int(x) for x in g["wide_cfg"])
    cell, wmin, wmax, shape = (float(x) for x in g["wide_fcfg"])
    spec = W.GridSpec(n_u, n_v, n_w, cell, w_min_native=wmin, w_max_native=wmax)
    kern = W.KernelSpec("gaussian", S, shape)
    u, v, w, t, vis, wt = chunk_from(g, "wide_in_")
    n = len(u)
    cuts = [0, n // 3, n // 2, n]
    batches = []
    for a, b in zip(cuts, cuts[1:]):
        batches.append(tuple(torch.from_numpy(np.ascontiguousarray(x[a:b])).pin_memory().numpy()
                             for x in (u, v, w, vis, wt)))
    got = list(W.image_stream(batches, spec, kern))
    assert len(got) == 3
    for bt, (img, d) in zip(batches, got):
        ref, dref = W.image(bt[0], bt[1], bt[2], None, bt[3], bt[4], spec, kern)
        assert img.pixels.tobytes() == ref.pixels.tobytes()
        assert img.imag_residual_norm == ref.imag_residual_norm
        assert d["grid_updates"] == dref["grid_updates"]


@pytest.mark.parametrize("name", ["small", "kb5", "kb1", "nw1", "wide", "multichan"])
def test_image_fp32_path_within_1e5(W, golden_image, name):
    """The optional FP32 path (complex64 grid and transforms, FP64
    coordinates / weights / phases / stack) against the reference image:
    north-star tolerance 1e-5 relative L2."""
    g = golden_image
    n_u, n_v, n_w, S, _ = (int(x) for x in g[f"{name}_cfg"])
    cell, wmin, wmax, shape = (float(x) for x in g[f"{name}_fcfg"])
    kind = "gaussian" if int(g[f"{name}_kind"][0]) == 0 else "kaiser_bessel"
    spec = W.GridSpec(n_u, n_v, n_w, cell, w_min_native=wmin, w_max_native=wmax)
    kern = W.KernelSpec(kind, S, shape)
    img, diag = W.image(*chunk_from(g, f"{name}_in_"), spec, kern, precision=32)
    assert diag["grid_updates"] == int(g[f"{name}_grid_updates"][0])
    err = rel_l2(img.pixels, g[f"{name}_pixels"])
    assert err <= 1e-5, err


def test_image_fp32_medium_and_device_path(W):
    """FP32 path on the 200k-record KB case vs the oracle, and through the
    device entry point (same kernels, same result)."""
    import torch
    src = ((0.02, -0.015, 2.0), (0.0, 0.0, 1.0), (-0.03, 0.01, 0.5))
    u, v, w, t, vis, wt = O.generate_synthetic(src, 200_000, 1, seed=21, cell_size_lm=5e-4,
                                               w_max_native=400.0)
    spec = W.GridSpec(256, 256, 8, 5e-4, w_max_native=400.0)
    kern = W.KernelSpec.kaiser_bessel(3)
    ref = O.image(u, v, w, t, vis, wt, 256, 256, 8, 5e-4, 0.0, 400.0, O.KIND_KAISER_BESSEL, 3,
                  kern.shape_param)
    img, _ = W.image(u, v, w, t, vis, wt, spec, kern, precision=32)
    assert rel_l2(img.pixels, ref["pixels"]) <= 1e-5
    dev = torch.device("cuda", 0)
    dimg, _ = W.image_device(*(torch.from_numpy(np.ascontiguousarray(x)).to(dev)
                               for x in (u, v, w, vis, wt)), spec, kern, precision=32)
    assert dimg.cpu().numpy().tobytes() == img.pixels.tobytes()
    # the context is back on FP64 afterwards
    d64, _ = W.image_device(*(torch.from_numpy(np.ascontiguousarray(x)).to(dev)
                              for x in (u, v, w, vis, wt)), spec, kern)
    assert rel_l2(d64.cpu().numpy(), ref["pixels"]) <= 1e-10


def test_linearity_complementary_halves(W):
    """Size-independent parity (the property run_cfg3.py --check applies at
    cfg3's full size): image(all) = image(A) + image(B) for complementary
    record halves A, B (other half's weights zeroed), and the update count
    does not depend on the weights."""
    import torch
    rng = np.random.default_rng(17)
    m = 1_000_000
    dev = torch.device("cuda", 0)
    u = torch.from_numpy(rng.uniform(0.1, 0.9, m)).to(dev)
    v = torch.from_numpy(rng.uniform(0.1, 0.9, m)).to(dev)
    w = torch.from_numpy(rng.uniform(0.0, 1.0, m)).to(dev)
    vis = torch.from_numpy((rng.standard_normal(m) + 1j * rng.standard_normal(m)).astype(np.complex64)).to(dev)
    wt = torch.from_numpy(rng.uniform(0.2, 1.0, m).astype(np.float32)).to(dev)
    spec = W.GridSpec(1024, 1024, 16, 2e-4, w_max_native=500.0)
    kern = W.KernelSpec.gaussian(3, 1.0)
    mask = torch.from_numpy(rng.random(m) < 0.5).to(dev)
    pall, dall = W.image_device(u, v, w, vis, wt, spec, kern)
    pall = pall.clone()
    pa, da = W.image_device(u, v, w, vis, torch.where(mask, wt, 0 * wt), spec, kern)
    pa = pa.clone()
    pb, db = W.image_device(u, v, w, vis, torch.where(mask, 0 * wt, wt), spec, kern)
    assert da["grid_updates"] == db["grid_updates"] == dall["grid_updates"]
    err = float((pall - pa - pb).norm() / pall.norm())
    assert err <= 1e-12, err
