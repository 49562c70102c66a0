"""Parity at the BASELINE configurations, GPU through the C ABI
against the pinned CPU oracle. Needs a B200.

* cfg1 (1M records, 512x512x8, Gaussian support 7, FP64; the reference's
  own CPU-runnable case): grid_updates = 35,789,105 (the reference's count at
  seed 1) and the whole image within 1e-10 relative L2.
* cfg2 (10M records, 2048x2048x32, the benched configuration):
  grid_updates = 359,470,496, the whole image within 1e-10
  of the oracle image, and one 128-row block of all 32 planes of the grid
  within 1e-12 max-abs of the slab-restricted oracle (grid_sector on one
  SectorBatch, gridder.py:186-204).
* cfg3 (100M LOFAR-like track records, 4096x4096x64, the north-star mesh):
  the grid rows around the densest anchor row (all 64 planes) against the
  slab-restricted oracle, and grid_updates against the closed-form count.
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_l2
from oracle import wstack_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SKY = ((0.02, -0.015, 2.0), (0.0, 0.0, 1.0))
THREADS = max(1, min(32, len(os.sched_getaffinity(0))))


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_00959_b200 as W
    return W


def _rel_max(a, b):
    """max |a - b| relative to max |b| (dense cells accumulate thousands of
    O(1) contributions, so the FP64 rounding of a different summation order
    scales with the cell magnitude)."""
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1.0))


def _synthetic(n, n_u, cell, seed=1):
    return O.generate_synthetic(SKY, n, 1, seed, cell_size_lm=cell, w_max_native=1000.0)


def test_cfg1_full_image_and_update_count(W):
    n, n_u, n_w, cell = 1_000_000, 512, 8, 1e-3
    u, v, w, t, vis, wt = _synthetic(n, n_u, cell)
    spec = W.GridSpec(n_u, n_u, n_w, cell, w_max_native=1000.0)
    kern = W.KernelSpec.gaussian(3, 1.0)
    img, diag = W.image(u, v, w, t, vis, wt, spec, kern)
    assert diag["grid_updates"] == 35_789_105
    ref = O.image(u, v, w, t, vis, wt, n_u, n_u, n_w, cell, 0.0, 1000.0, O.KIND_GAUSSIAN, 3, 1.0,
                  threads=THREADS)
    assert ref["grid_updates"] == 35_789_105
    err = rel_l2(img.pixels, ref["pixels"])
    assert err <= 1e-10, err
    np.testing.assert_allclose([img.imag_residual_norm, img.real_norm],
                               [ref["imag_residual_norm"], ref["real_norm"]], rtol=1e-9)


@pytest.fixture(scope="module")
def cfg2(W):
    n, n_u, n_w, cell = 10_000_000, 2048, 32, 2e-4
    u, v, w, t, vis, wt = _synthetic(n, n_u, cell)
    spec = W.GridSpec(n_u, n_u, n_w, cell, w_max_native=1000.0)
    return spec, (u, v, w, t, vis, wt)


@pytest.mark.parametrize("slabs", [1, 3])
def test_cfg2_bucketing_bitexact(W, cfg2, slabs):
    """K1 (wsb_bucket_items) at the benched size: every (record, work item)
    entry, its key and the item order equal the restated contract
    (oracle.item_entries, taps of gridder.py:164-177), for the whole mesh and
    for a slab of an uneven 3-way split."""
    spec, (u, v, w, t, vis, wt) = cfg2
    dev = torch.device("cuda", 0)
    rec, plane = W.prepare_device(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                                    for a in (u, v, w, vis, wt)), spec)
    v0, vc = (0, spec.n_v) if slabs == 1 else (700, 650)
    gv = rec[:, 1].cpu().numpy()
    sel = np.nonzero(O.halo_mask(gv, 3, v0, vc))[0]
    r = rec[torch.from_numpy(sel).to(dev)].contiguous()
    pl = plane[torch.from_numpy(sel).to(dev)].contiguous()
    keys, idx, off, ib = W.bucket_items_device(r, pl, spec, 3, v0, vc)
    from paper_2504_00959_b200 import _lib as L
    rk, ri, ro, rib = O.item_entries(u[sel] * spec.n_u, v[sel] * spec.n_v,
                                     O.plane_of_w(w[sel], spec.n_w), spec.n_u, spec.n_w, 3, v0, vc,
                                     ss_cols=L.ITEM_COLS)
    assert ib == rib
    assert np.array_equal(off, ro)
    assert np.array_equal(keys, rk)
    assert np.array_equal(idx, ri)


def test_cfg2_update_count_and_grid_block(W, cfg2):
    spec, (u, v, w, t, vis, wt) = cfg2
    kern = W.KernelSpec.gaussian(3, 1.0)
    dev = torch.device("cuda", 0)
    rec, plane = W.prepare_device(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                                    for a in (u, v, w, vis, wt)), spec)
    gs, upd = W.grid_slab_device(rec, plane, spec, kern, 0, spec.n_v)
    assert upd == 359_470_496
    prep = O.prepare(u, v, w, t, vis, wt, spec.n_u, spec.n_v, spec.n_w)
    prep.update(v_start=0, v_count=spec.n_v)
    for r0 in (0, 960, spec.n_v - 128):      # both mesh edges and an interior block
        got = W.unpack_grid_device(gs, spec, 0, spec.n_v, rows=(r0, r0 + 128)).cpu().numpy()
        ref, _ = O.grid_rows(prep, spec.n_u, spec.n_w, O.KIND_GAUSSIAN, 3, 1.0, r0, r0 + 128)
        err = float(np.max(np.abs(got - ref)))
        assert err <= 1e-12, (r0, err)


def test_cfg2_full_image(W, cfg2):
    spec, (u, v, w, t, vis, wt) = cfg2
    kern = W.KernelSpec.gaussian(3, 1.0)
    img, diag = W.image(u, v, w, t, vis, wt, spec, kern)
    assert diag["grid_updates"] == 359_470_496
    ref = O.image(u, v, w, t, vis, wt, spec.n_u, spec.n_v, spec.n_w, spec.cell_size_lm, 0.0,
                  1000.0, O.KIND_GAUSSIAN, 3, 1.0, threads=THREADS)
    err = rel_l2(img.pixels, ref["pixels"])
    assert err <= 1e-10, err


def test_cfg3_densest_rows_vs_slab_restricted_oracle(W):
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    from lofar import tracks
    n, n_u, n_w, cell = 100_000_000, 4096, 64, 1e-4
    dev = torch.device("cuda", 0)
    u, v, w, t, vis, wt = tracks(n, cell, device=dev)
    spec = W.GridSpec(n_u, n_u, n_w, cell, w_max_native=1000.0)
    kern = W.KernelSpec.gaussian(3, 1.0)
    rec, plane = W.prepare_device(u, v, w, vis, wt, spec)
    gs, upd = W.grid_slab_device(rec, plane, spec, kern, 0, spec.n_v)
    del rec, plane
    gv = (v * n_u).cpu().numpy()           # exact: power-of-two scale
    hist = np.bincount(np.floor(gv).astype(np.int64), minlength=n_u)
    dense = int(np.argmax(hist))
    r0, r1 = dense - 8, dense + 8
    got = W.unpack_grid_device(gs, spec, 0, spec.n_v, rows=(r0, r1)).cpu().numpy()
    del gs
    torch.cuda.empty_cache()
    # the records that can reach the rows (halo predicate), in record order
    m = O.halo_mask(gv, 3, r0, r1 - r0)
    sel = torch.from_numpy(np.nonzero(m)[0]).to(dev)
    cols = [a[sel].cpu().numpy() for a in (u, v, w, t, vis, wt)]
    gu_all = (u * n_u).cpu().numpy()
    assert upd == O.count_updates(gu_all, gv, n_u, 0, n_u, 3)
    prep = O.prepare(*cols, n_u, n_u, n_w)
    prep.update(v_start=r0, v_count=r1 - r0)
    ref, cnt = O.grid_slab(prep, n_u, n_w, O.KIND_GAUSSIAN, 3, 1.0)
    assert cnt == O.count_updates(prep["gu"], prep["gv"], n_u, r0, r1, 3)
    assert len(cols[0]) > 1_000_000               # a dense band of the tracks
    err = _rel_max(got, ref)
    assert err <= 1e-12, err


def test_unsorted_time_index_raises_like_partition_time_ordered(W):
    """visdata.py:354-355 (reached by run_pipeline, pipeline.py:47-52):
    records must be sorted by time_index; sorted input is accepted."""
    u, v, w, t, vis, wt = O.generate_synthetic(SKY, 5000, 1, 3, cell_size_lm=1e-3,
                                               w_max_native=10.0)
    spec = W.GridSpec(64, 64, 4, 1e-3, w_max_native=10.0)
    kern = W.KernelSpec.gaussian(3, 1.0)
    ok, _ = W.image(u, v, w, t, vis, wt, spec, kern)
    bad = t.copy()
    bad[100], bad[4000] = bad[4000], bad[100]
    with pytest.raises(ValueError, match="sorted by time_index"):
        W.image(u, v, w, bad, vis, wt, spec, kern)
    same, _ = W.image(u, v, w, None, vis, wt, spec, kern)   # no time index: array order
    assert same.pixels.tobytes() == ok.pixels.tobytes()
