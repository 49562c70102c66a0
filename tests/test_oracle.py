"""Pin the CPU oracle against fixtures produced by the reference itself
(tests/golden/make_golden.py). CPU only."""

import numpy as np
import pytest

from conftest import chunk_from, rel_l2
from oracle import wstack_oracle as O


def _parts(u, v, w, t, vis, wt, R, n_u, n_v, n_w):
    """partition_time_ordered (visdata.py:344-366) + prepare per part."""
    slices = np.unique(t)
    parts, off = [], 0
    for r in range(R):
        s0, sc = O.partition_1d(len(slices), R, r)
        lo = np.searchsorted(t, slices[s0], side="left")
        hi = np.searchsorted(t, slices[s0 + sc - 1], side="right")
        parts.append(O.prepare(u[lo:hi], v[lo:hi], w[lo:hi], t[lo:hi], vis[lo:hi], wt[lo:hi],
                               n_u, n_v, n_w, gindex_offset=off))
        off += hi - lo
    return parts


@pytest.mark.parametrize("name", ["syn", "edge"])
def test_prepare_bitexact(golden_bucket, name):
    g = golden_bucket
    n_u, n_v, n_w, S = (int(x) for x in g[f"{name}_spec"])
    prep = O.prepare(*chunk_from(g, f"{name}_in_"), n_u, n_v, n_w)
    for k in ("gu", "gv", "plane", "gindex"):
        assert np.array_equal(prep[k], g[f"{name}_prep_{k}"]), k
    assert prep["value"].tobytes() == g[f"{name}_prep_value"].tobytes()


@pytest.mark.parametrize("name", ["syn", "edge"])
@pytest.mark.parametrize("R", [1, 2, 4, 8])
def test_exchange_bitexact(golden_bucket, name, R):
    g = golden_bucket
    n_u, n_v, n_w, S = (int(x) for x in g[f"{name}_spec"])
    parts = _parts(*chunk_from(g, f"{name}_in_"), R, n_u, n_v, n_w)
    batches = O.exchange(parts, n_v, R, S)
    for d, b in enumerate(batches):
        for col in ("gu", "gv", "plane", "value", "time_index", "gindex", "is_halo"):
            ref = g[f"{name}_R{R}_d{d}_{col}"]
            assert b[col].tobytes() == ref.astype(b[col].dtype).tobytes(), (d, col)


@pytest.mark.parametrize("kname", ["gauss3", "gauss1", "kb1", "kb3", "kb5"])
def test_grid_bitexact(golden_grid, kname):
    g = golden_grid
    n_u = n_v = 64
    n_w = 4
    S = int(g[f"{kname}_S"][0])
    shape = float(g[f"{kname}_shape"][0])
    kind = O.KIND_GAUSSIAN if kname.startswith("gauss") else O.KIND_KAISER_BESSEL
    prep = O.prepare(*chunk_from(g, "in_"), n_u, n_v, n_w)
    grid, updates = O.grid_all([prep], n_u, n_v, n_w, kind, S, shape, 1)
    assert updates == int(g[f"{kname}_updates"][0])
    assert grid.tobytes() == g[f"{kname}_grid"].tobytes()


@pytest.mark.parametrize("name", ["small", "kb5", "kb1", "nw1", "wide", "multichan"])
def test_image_matches_reference(golden_image, name):
    g = golden_image
    n_u, n_v, n_w, S, ranks = (int(x) for x in g[f"{name}_cfg"])
    cell, wmin, wmax, shape = (float(x) for x in g[f"{name}_fcfg"])
    kind = int(g[f"{name}_kind"][0])
    res = O.image(*chunk_from(g, f"{name}_in_"), n_u, n_v, n_w, cell, wmin, wmax,
                  kind=kind, half_support=S, shape=shape)
    assert res["grid_updates"] == int(g[f"{name}_grid_updates"][0])
    assert rel_l2(res["pixels"], g[f"{name}_pixels"]) <= 1e-12
    np.testing.assert_allclose([res["imag_residual_norm"], res["real_norm"]],
                               g[f"{name}_norms"], rtol=1e-10, atol=1e-300)


def test_threaded_oracle_bit_identical(golden_image):
    g = golden_image
    n_u, n_v, n_w, S, _ = (int(x) for x in g["wide_cfg"])
    cell, wmin, wmax, shape = (float(x) for x in g["wide_fcfg"])
    a = O.image(*chunk_from(g, "wide_in_"), n_u, n_v, n_w, cell, wmin, wmax, 0, S, shape, threads=1)
    b = O.image(*chunk_from(g, "wide_in_"), n_u, n_v, n_w, cell, wmin, wmax, 0, S, shape, threads=4)
    assert a["grid"].tobytes() == b["grid"].tobytes()
    assert a["grid_updates"] == b["grid_updates"]


def test_validation_errors():
    with pytest.raises(ValueError):
        O.validate_grid(48, 64, 4, 1e-3)
    with pytest.raises(ValueError):
        O.validate_grid(64, 64, 0, 1e-3)
    with pytest.raises(ValueError):
        O.validate_grid(4096, 4096, 4, 1e-3)   # FoV too wide
    with pytest.raises(ValueError):
        O.prepare([1.0], [0.5], [0.5], [0], [[1 + 0j]], [[1.0]], 8, 8, 2)
    with pytest.raises(ValueError):
        O.prepare([0.5], [0.5], [1.5], [0], [[1 + 0j]], [[1.0]], 8, 8, 2)
    with pytest.raises(ValueError):
        O.prepare([0.5], [0.5], [0.5], [0], [[1 + 0j]], [[-1.0]], 8, 8, 2)


def test_item_entries_cover_every_update(golden_grid):
    """The gridder's work-item bucketing restated (oracle.item_entries): the
    per-entry tap products add up to the reference's grid_updates, every
    record with taps in the slab appears, and items are in record order."""
    g = golden_grid
    for R in (1, 2, 3):
        tot = 0
        n_u, n_v = 64, 96
        rng = np.random.default_rng(7)
        gu, gv = rng.uniform(0, n_u, 3000), rng.uniform(0, n_v, 3000)
        gu[:5] = [0.0, 63.5, 31.0, 64 - 1e-9, 2.999]          # edges, integers
        plane = rng.integers(0, 3, 3000)
        for d in range(R):
            v0, vc = O.partition_1d(n_v, R, d)
            m = O.halo_mask(gv, 3, v0, vc)
            keys, idx, off, ib = O.item_entries(gu[m], gv[m], plane[m], n_u, 3, 3, v0, vc,
                                                ss_cols=16, item_rows=8)
            assert np.all(np.diff(keys.astype(np.int64)) >= 0)
            same = np.diff(keys.astype(np.int64)) == 0     # equal keys: record order
            assert np.all(np.diff(idx.astype(np.int64))[same] > 0)
            n_rb = -(-vc // 8)
            for k, i in zip(keys, idx):
                item = int(k) >> 8
                rb, ss = item % n_rb, (item // n_rb) % 4
                c0, c1 = O.tap_bounds(gu[m][i:i + 1], 3, ss * 16, ss * 16 + 15)
                r0, r1 = O.tap_bounds(gv[m][i:i + 1], 3, v0 + rb * 8, min(v0 + rb * 8 + 7, v0 + vc - 1))
                assert c0[0] <= c1[0] and r0[0] <= r1[0]
                tot += int((c1[0] - c0[0] + 1) * (r1[0] - r0[0] + 1))
        assert tot == O.count_updates(gu, gv, n_u, 0, n_v, 3)
