"""CPU oracle for the w-stacking hot path — TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference ``wstack`` package's
imaging hot path (``/root/reference/pkg/src/wstack``).  It exists to check
the CUDA product path; only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product package ``paper_2504_00959_b200`` never imports it and has no
CPU fallback.

Parity is PINNED: ``tests/golden/make_golden.py`` runs the reference itself
(imported read-only from ``/root/reference``) and stores its outputs under
``tests/golden/*.npz``; ``tests/test_oracle.py`` checks this module against
those fixtures (bucketing bit-exact, grids bit-exact in the reference's
tap-major accumulation order, images to <= 1e-12 relative L2 because the
FFT here is pocketfft instead of the reference's radix-2 loop).

Every function cites the reference lines it restates.
"""

from __future__ import annotations

import concurrent.futures as _cf
import math

import numpy as np

KIND_GAUSSIAN = 0
KIND_KAISER_BESSEL = 1
DEFAULT_KB_BETA_PER_SUPPORT = 2.34          # gridder.py:44


# ---------------------------------------------------------------------------
# geometry (mesh.py)
# ---------------------------------------------------------------------------

def partition_1d(n: int, parts: int, index: int):
    """Balanced contiguous split (mesh.py:34-45). Returns (start, count)."""
    if parts < 1 or not (0 <= index < parts):
        raise ValueError(f"invalid partition index {index} of {parts}")
    q, r = divmod(n, parts)
    if index < r:
        return index * (q + 1), q + 1
    return r * (q + 1) + (index - r) * q, q


def slabs(n_v: int, n_ranks: int):
    """[(v_start, v_count)] per rank (mesh.py:152-159)."""
    if n_ranks > n_v:
        raise ValueError(f"n_ranks {n_ranks} exceeds n_v {n_v}")
    return [partition_1d(n_v, n_ranks, r) for r in range(n_ranks)]


def plane_of_w(w: np.ndarray, n_w: int) -> np.ndarray:
    """Nearest plane, half up, clipped (comms.py:484-488, mesh.py:162-167)."""
    if n_w == 1:
        return np.zeros(len(w), dtype=np.uint32)
    k = np.floor(w * (n_w - 1) + 0.5).astype(np.int64)
    return np.clip(k, 0, n_w - 1).astype(np.uint32)


def plane_w_native(k: int, n_w: int, w_min_native: float, w_max_native: float) -> float:
    """Native w of plane k; midpoint for a single plane (mesh.py:101-112)."""
    if n_w == 1:
        return 0.5 * (w_min_native + w_max_native)
    frac = k / (n_w - 1)
    return w_min_native + frac * (w_max_native - w_min_native)


def validate_grid(n_u, n_v, n_w, cell_size_lm, w_min_native=0.0, w_max_native=0.0):
    """GridSpec.__post_init__ rules (mesh.py:79-95)."""
    def pow2(n):
        return n >= 1 and (n & (n - 1)) == 0
    if n_u < 2 or not pow2(n_u):
        raise ValueError(f"n_u must be a power of two >= 2, got {n_u}")
    if n_v < 2 or not pow2(n_v):
        raise ValueError(f"n_v must be a power of two >= 2, got {n_v}")
    if n_w < 1:
        raise ValueError(f"n_w must be >= 1, got {n_w}")
    if cell_size_lm <= 0.0:
        raise ValueError("cell_size_lm must be positive")
    half_l = n_u * cell_size_lm / 2.0
    half_m = n_v * cell_size_lm / 2.0
    if half_l >= 1.0 or half_m >= 1.0 or half_l * half_l + half_m * half_m >= 1.0:
        raise ValueError("field of view too wide: corner pixels leave the unit disc")
    if w_min_native > w_max_native:
        raise ValueError("w_min_native must be <= w_max_native")


# ---------------------------------------------------------------------------
# record preparation + exchange (comms.py)
# ---------------------------------------------------------------------------

def validate_chunk(u, v, w, weight):
    """VisChunk.validate (visdata.py:178-184)."""
    if np.any(u < 0) or np.any(u >= 1) or np.any(v < 0) or np.any(v >= 1):
        raise ValueError("u and v must lie in [0, 1)")
    if np.any(w < 0) or np.any(w > 1):
        raise ValueError("w must lie in [0, 1]")
    if not np.all(np.isfinite(weight)) or np.any(weight < 0):
        raise ValueError("weights must be finite and >= 0")


def prepare(u, v, w, time_index, vis, weight, n_u, n_v, n_w, gindex_offset=0):
    """prepare_chunk (comms.py:477-492): gu, gv, plane, time, gindex, value.

    ``value`` is the complex128 product vis*weight summed over channels in
    NumPy's own reduction order (pairwise for >= 4 channels)."""
    u = np.ascontiguousarray(u, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    w = np.ascontiguousarray(w, np.float64)
    vis = np.ascontiguousarray(np.atleast_2d(vis), np.complex64)
    weight = np.ascontiguousarray(np.atleast_2d(weight), np.float32)
    validate_chunk(u, v, w, weight)
    n = len(u)
    return {
        "gu": u * n_u,
        "gv": v * n_v,
        "plane": plane_of_w(w, n_w),
        "time_index": np.ascontiguousarray(time_index, np.uint32),
        "gindex": np.uint64(gindex_offset) + np.arange(n, dtype=np.uint64),
        "value": (vis.astype(np.complex128) * weight).sum(axis=1),
    }


def halo_mask(gv: np.ndarray, halo_rows: int, v_start: int, v_count: int) -> np.ndarray:
    """Destination test of the time->space exchange (comms.py:521-523)."""
    return (gv + halo_rows >= v_start) & (gv - halo_rows <= v_start + v_count - 1)


def exchange(prepared_parts, n_v: int, n_ranks: int, halo_rows: int):
    """exchange_to_space_order (comms.py:495-547) without the message log.

    ``prepared_parts`` is one ``prepare`` dict per source rank (gindex
    offsets already applied). Returns one batch dict per destination slab,
    rows sorted by (time_index, gindex), with ``is_halo``."""
    out = []
    for d, (v0, vc) in enumerate(slabs(n_v, n_ranks)):
        cols = {k: [] for k in ("gu", "gv", "plane", "time_index", "gindex", "value")}
        # own part first, then the others in rank order (comms.py:525-531);
        # the lexsort below makes the arrival order irrelevant.
        order = [d] + [s for s in range(n_ranks) if s != d]
        for s in order:
            p = prepared_parts[s]
            m = halo_mask(p["gv"], halo_rows, v0, vc)
            for k in cols:
                cols[k].append(p[k][m])
        cat = {k: np.concatenate(cols[k]) for k in cols}
        srt = np.lexsort((cat["gindex"], cat["time_index"]))
        cat = {k: cat[k][srt] for k in cat}
        rows = np.floor(cat["gv"]).astype(np.int64)
        cat["is_halo"] = ~((rows >= v0) & (rows < v0 + vc))
        cat["v_start"] = v0
        cat["v_count"] = vc
        out.append(cat)
    return out


# ---------------------------------------------------------------------------
# gridding kernel + scatter (gridder.py)
# ---------------------------------------------------------------------------

def default_shape_param(kind: int, half_support: int) -> float:
    """KernelSpec.gaussian sigma=1 / kaiser_bessel beta=2.34*S (gridder.py:64-72)."""
    return 1.0 if kind == KIND_GAUSSIAN else DEFAULT_KB_BETA_PER_SUPPORT * half_support


def _kb_axis(S: int, beta: float, x):
    """Kaiser-Bessel axis factor (gridder.py:92-98)."""
    Sf = float(S)
    inside = np.abs(x) <= Sf
    t = np.where(inside, 1.0 - (x / Sf) ** 2, 0.0)
    vals = np.i0(beta * np.sqrt(t)) / np.i0(beta)
    return np.where(inside, vals, 0.0)


def kernel_value(kind: int, S: int, shape: float, du, dv):
    """Unit-peak Gaussian / separable Kaiser-Bessel (gridder.py:75-89)."""
    du = np.asarray(du, dtype=np.float64)
    dv = np.asarray(dv, dtype=np.float64)
    if kind == KIND_GAUSSIAN:
        s2 = 2.0 * shape * shape
        return np.exp(-(du * du + dv * dv) / s2)
    return _kb_axis(S, shape, du) * _kb_axis(S, shape, dv)


def grid_slab(batch, n_u: int, n_w: int, kind: int, S: int, shape: float,
              row_lo: int | None = None, row_hi: int | None = None):
    """_accumulate (gridder.py:160-183) for one slab, tap-major order.

    Returns (grid[n_w, v_count, n_u] complex128, grid_updates)."""
    v0, vc = batch["v_start"], batch["v_count"]
    row_lo = v0 if row_lo is None else row_lo
    row_hi = v0 + vc if row_hi is None else row_hi
    out = np.zeros((n_w, vc, n_u), dtype=np.complex128)
    gu, gv, value = batch["gu"], batch["gv"], batch["value"]
    if len(gu) == 0:
        return out, 0
    if np.any(gv + S < v0) or np.any(gv - S > v0 + vc - 1):          # gridder.py:198-199
        raise ValueError("record outside slab+halo")
    flo_u = np.floor(gu).astype(np.int64)
    flo_v = np.floor(gv).astype(np.int64)
    pl = batch["plane"].astype(np.int64)
    count = 0
    for a in range(-S, S + 1):
        i = flo_u + a
        du = gu - i
        ok_u = (np.abs(du) <= S) & (i >= 0) & (i < n_u)
        if not ok_u.any():
            continue
        for b in range(-S, S + 1):
            j = flo_v + b
            dv = gv - j
            ok = ok_u & (np.abs(dv) <= S) & (j >= row_lo) & (j < row_hi)
            if not ok.any():
                continue
            kv = kernel_value(kind, S, shape, du[ok], dv[ok])
            np.add.at(out, (pl[ok], j[ok] - v0, i[ok]), value[ok] * kv)
            count += int(ok.sum())
    return out, count


def select_rows(batch, S: int, row_lo: int, row_hi: int):
    """The records of ``batch`` whose footprint can reach rows
    [row_lo, row_hi): the halo predicate of comms.py:521-523 applied to a
    row block instead of a rank's slab. Record order is kept, so gridding
    the selection reproduces those rows of the full slab bit for bit (every
    tap pass of _accumulate visits the surviving records in the same order).
    Returns a batch dict with v_start = row_lo, v_count = row_hi - row_lo."""
    m = halo_mask(batch["gv"], S, row_lo, row_hi - row_lo)
    out = {k: batch[k][m] for k in ("gu", "gv", "plane", "value")}
    out["v_start"], out["v_count"] = row_lo, row_hi - row_lo
    return out


def grid_rows(batch, n_u: int, n_w: int, kind: int, S: int, shape: float,
              row_lo: int, row_hi: int):
    """Rows [row_lo, row_hi) of the slab grid of ``batch`` (the slab-restricted
    oracle of SURVEY 8c: grid_sector on one SectorBatch, gridder.py:186-204),
    without materialising the rest of the slab. Returns
    (grid[n_w, row_hi - row_lo, n_u], grid_updates inside the rows)."""
    return grid_slab(select_rows(batch, S, row_lo, row_hi), n_u, n_w, kind, S, shape)


def count_updates(gu, gv, n_u: int, row_lo: int, row_hi: int, S: int) -> int:
    """grid_sector's update count (gridder.py:164-183, 259) in closed form:
    per record, (#columns i with |gu-i| <= S, 0 <= i < n_u) x (#rows j with
    |gv-j| <= S, row_lo <= j < row_hi); the tap tests are the reference's."""
    gu = np.asarray(gu, np.float64)
    gv = np.asarray(gv, np.float64)
    total = 0
    step = 1 << 22
    for a0 in range(0, len(gu), step):
        cu = np.zeros(len(gu[a0:a0 + step]), np.int64)
        cv = np.zeros_like(cu)
        fu, fv = np.floor(gu[a0:a0 + step]), np.floor(gv[a0:a0 + step])
        for a in range(-S, S + 1):
            i = fu + a
            cu += (np.abs(gu[a0:a0 + step] - i) <= S) & (i >= 0) & (i < n_u)
            j = fv + a
            cv += (np.abs(gv[a0:a0 + step] - j) <= S) & (j >= row_lo) & (j < row_hi)
        total += int((cu * cv).sum())
    return total


def tap_bounds(g, S: int, lo: int, hi: int):
    """First / last tap index {i : |g - i| <= S} (gridder.py:164-177) clipped
    to [lo, hi], per record (empty where first > last)."""
    g = np.asarray(g, np.float64)
    fl = np.floor(g).astype(np.int64)
    i0 = fl - S
    i0 = np.where(g - i0 > S, i0 + 1, i0)
    return np.maximum(i0, lo), np.minimum(fl + S, hi)


def item_entries(gu, gv, plane, n_u: int, n_w: int, S: int, v_start: int, v_count: int,
                 ss_cols: int = 16, item_rows: int = 128, row_bits: int = 8):
    """The GPU gridder's work-item bucketing restated (contract of
    wsb_bucket_items, include/wsb.h): every (record, item) pair whose taps
    reach item = (plane, ss_cols-column block, item_rows-row block of
    the slab), key = item << row_bits | rowrel with rowrel = floor(gv) - S -
    (block row0 - 2S), stably sorted by key (record order for equal keys).
    Tap sets are the reference's (gridder.py:164-177). Returns
    (keys u32, idx u32, off u32[n_items + 1], item_bits)."""
    gu, gv = np.asarray(gu, np.float64), np.asarray(gv, np.float64)
    plane = np.asarray(plane, np.int64)
    n_ss = -(-n_u // ss_cols)
    n_rb = -(-v_count // item_rows)
    n_items = n_w * n_ss * n_rb
    item_bits = max(1, int(np.ceil(np.log2(n_items))) if n_items > 1 else 0)
    i0, i1 = tap_bounds(gu, S, 0, n_u - 1)
    j0, j1 = tap_bounds(gv, S, v_start, v_start + v_count - 1)
    ok = (i0 <= i1) & (j0 <= j1)
    anchor = np.floor(gv).astype(np.int64) - S
    keys, idx = [], []
    rec = np.arange(len(gu), dtype=np.int64)
    for drb in (0, 1):
        for dss in (0, 1):
            ss = i0 // ss_cols + dss
            rb = (j0 - v_start) // item_rows + drb
            m = ok & (ss <= i1 // ss_cols) & (rb <= (j1 - v_start) // item_rows)
            item = (plane[m] * n_ss + ss[m]) * n_rb + rb[m]
            rowrel = anchor[m] - (v_start + rb[m] * item_rows - 2 * S)
            keys.append(((item << row_bits) | rowrel).astype(np.uint32))
            idx.append(rec[m])
    keys, idx = np.concatenate(keys), np.concatenate(idx)
    order = np.lexsort((idx, keys))           # by key, then record
    keys, idx = keys[order], idx[order].astype(np.uint32)
    cnt = np.bincount(keys >> row_bits, minlength=n_items)
    off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint32)
    return keys, idx, off, item_bits


def grid_all(prepared_parts, n_u, n_v, n_w, kind, S, shape, n_ranks):
    """grid_all (gridder.py:262-294): exchange then grid each slab; the
    reduce is the identity after the exchange (pipeline.py:117-122).
    Returns (full grid (n_w, n_v, n_u), total grid_updates)."""
    batches = exchange(prepared_parts, n_v, n_ranks, S)
    grids, total = [], 0
    for b in batches:
        g, c = grid_slab(b, n_u, n_w, kind, S, shape)
        grids.append(g)
        total += c
    return np.concatenate(grids, axis=1), total


# ---------------------------------------------------------------------------
# transform, w correction, stacking (transform.py)
# ---------------------------------------------------------------------------

def checker_sign(n_u: int, v_start: int, v_count: int) -> np.ndarray:
    """(-1)^(i+j) (transform.py:180-185)."""
    i = np.arange(n_u, dtype=np.int64)
    j = np.arange(v_start, v_start + v_count, dtype=np.int64)
    return (1.0 - 2.0 * ((i[None, :] + j[:, None]) & 1)).astype(np.float64)


def ifft2(plane: np.ndarray) -> np.ndarray:
    """Inverse 2D DFT, e^{+2 pi i}, scaled 1/(n_u n_v) (transform.py:99-127).
    pocketfft instead of the reference's radix-2 loop (<= 1e-15 relative)."""
    return np.fft.ifft2(plane)


def pixel_lm(n_u, n_v, cell, v_start, v_count):
    """pixel_lm_blocks (mesh.py:202-208)."""
    cols = np.arange(n_u, dtype=np.float64) - n_u // 2
    rows = np.arange(v_start, v_start + v_count, dtype=np.float64) - n_v // 2
    l = np.broadcast_to(cols * cell, (v_count, n_u))
    m = np.broadcast_to((rows * cell)[:, None], (v_count, n_u))
    return l, m


def w_correct(plane, k, n_u, n_v, n_w, cell, w_min_native, w_max_native, v_start, v_count):
    """apply_w_correction (transform.py:192-202)."""
    w_k = plane_w_native(k, n_w, w_min_native, w_max_native)
    if w_k == 0.0:
        return plane.copy()
    l, m = pixel_lm(n_u, n_v, cell, v_start, v_count)
    n = np.sqrt(1.0 - l * l - m * m)
    return plane * np.exp(2j * np.pi * w_k * (n - 1.0))


def stack(planes, n_u, n_v, n_w, cell, v_start, v_count):
    """stack_planes (transform.py:205-230). Returns (pixels, imag_sq, real_sq)."""
    acc = planes[0].astype(np.complex128, copy=True)
    for p in planes[1:]:
        acc = acc + p
    acc /= n_w
    l, m = pixel_lm(n_u, n_v, cell, v_start, v_count)
    acc *= np.sqrt(1.0 - l * l - m * m)
    return (np.ascontiguousarray(acc.real), float((acc.imag ** 2).sum()),
            float((acc.real ** 2).sum()))


def image_from_grid(grid, n_u, n_v, n_w, cell, w_min_native, w_max_native, threads=1):
    """Phases fft + wcorrect + write of run_pipeline (pipeline.py:125-152)
    on a full (single-slab) grid. ``threads`` > 1 transforms and corrects
    planes concurrently (the planes are independent, pipeline.py:127-147);
    the stack still sums them in plane order. Returns (pixels, imag_norm,
    real_norm)."""
    sign = checker_sign(n_u, 0, n_v)

    def plane(k):
        p = ifft2(grid[k] * sign)
        return w_correct(p, k, n_u, n_v, n_w, cell, w_min_native, w_max_native, 0, n_v)

    if threads > 1:
        with _cf.ThreadPoolExecutor(threads) as ex:
            planes = list(ex.map(plane, range(n_w)))
    else:
        planes = [plane(k) for k in range(n_w)]
    pix, isq, rsq = stack(planes, n_u, n_v, n_w, cell, 0, n_v)
    return pix, math.sqrt(isq), math.sqrt(rsq)


def image(u, v, w, time_index, vis, weight, n_u, n_v, n_w, cell, w_min_native,
          w_max_native, kind=KIND_GAUSSIAN, half_support=3, shape=None, threads=1):
    """Dirty image through the reference's hot path (pipeline.py:95-152).

    ``threads`` > 1 grids row blocks of the single slab concurrently, the
    reference's deterministic threaded mode (gridder.py:206-221), so the
    grid is bit-identical for any thread count.
    Returns dict(pixels, imag_residual_norm, real_norm, grid_updates)."""
    validate_grid(n_u, n_v, n_w, cell, w_min_native, w_max_native)
    if shape is None:
        shape = default_shape_param(kind, half_support)
    prep = prepare(u, v, w, time_index, vis, weight, n_u, n_v, n_w, 0)
    batch = exchange([prep], n_v, 1, half_support)[0]
    if threads <= 1:
        grid, updates = grid_slab(batch, n_u, n_w, kind, half_support, shape)
    else:
        grid = np.zeros((n_w, n_v, n_u), np.complex128)
        # row blocks as the reference's deterministic threads (gridder.py:206-221);
        # each thread holds only its block (grid_rows), not a whole slab
        blocks = [partition_1d(n_v, threads, t) for t in range(threads)]

        def work(blk):
            b0, bc = blk
            g, c = grid_rows(batch, n_u, n_w, kind, half_support, shape, b0, b0 + bc)
            grid[:, b0:b0 + bc] = g
            return c

        with _cf.ThreadPoolExecutor(threads) as ex:
            updates = sum(ex.map(work, blocks))
    pix, inorm, rnorm = image_from_grid(grid, n_u, n_v, n_w, cell, w_min_native, w_max_native,
                                        threads)
    return {"pixels": pix, "imag_residual_norm": inorm, "real_norm": rnorm,
            "grid_updates": updates, "grid": grid}


# ---------------------------------------------------------------------------
# synthetic data (visdata.py:369-434) — the generator both arms are fed from
# ---------------------------------------------------------------------------

def point_source_visibility(sources, u_native, v_native, w_native):
    """visdata.py:369-381."""
    out = np.zeros(np.shape(u_native), dtype=np.complex128)
    for l, m, flux in sources:
        n = np.sqrt(1.0 - l * l - m * m)
        phase = -2.0 * np.pi * (u_native * l + v_native * m + w_native * (n - 1.0))
        out += (flux / n) * np.exp(1j * phase)
    return out


def generate_synthetic(sources, n_records, n_freq, seed, n_time_slices=8,
                       cell_size_lm=1e-3, w_min_native=0.0, w_max_native=0.0, n_corr=1):
    """generate_synthetic (visdata.py:384-434): PCG64 uniform uvw, exact
    point-source visibilities, unit weights."""
    rng = np.random.default_rng(seed)
    u = rng.random(n_records)
    v = rng.random(n_records)
    w = rng.random(n_records)
    time_index = (np.arange(n_records, dtype=np.uint64) * n_time_slices
                  // n_records).astype(np.uint32)
    value = point_source_visibility(sources, u / cell_size_lm, v / cell_size_lm,
                                    w_min_native + w * (w_max_native - w_min_native))
    n_chan = n_freq * n_corr
    vis = np.repeat(value.astype(np.complex64)[:, None], n_chan, axis=1)
    weight = np.ones((n_records, n_chan), dtype=np.float32)
    return u, v, w, time_index, vis, weight
