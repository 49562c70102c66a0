"""LOFAR-like synthetic uv tracks (BASELINE config 3): earth-rotation
tracks of a core-heavy station layout, time-sorted, normalised into [0, 1)
around u = v = 0.5 so the reference's conventions apply (u_native = u / cell,
visdata.py:419-424; w affine onto [w_min_native, w_max_native]).

Values are point-source visibilities evaluated like
visdata.point_source_visibility (visdata.py:369-381), in FP64 on the GPU;
weights are 1. Returns torch tensors on ``device``.
"""

from __future__ import annotations

import math

import numpy as np
import torch

SOURCES = ((0.02, -0.015, 2.0), (0.0, 0.0, 1.0), (-0.05, 0.03, 0.5))


def tracks(n_records: int, cell: float, w_max_native: float = 1000.0, n_stations: int = 62,
           n_time_slices: int = 8, seed: int = 3, dec_deg: float = 52.0, max_uv_frac: float = 0.45,
           sources=SOURCES, device="cuda", first: int = 0, count: int | None = None):
    """Records [first, first+count) of the full time-ordered track set (a
    rank's time partition)."""
    rng = np.random.default_rng(seed)
    n_core = n_stations // 2
    core = rng.normal(0.0, 0.02, (n_core, 2))
    r = np.exp(rng.uniform(np.log(0.05), np.log(1.0), n_stations - n_core))
    th = rng.uniform(0, 2 * np.pi, n_stations - n_core)
    arms = np.stack([r * np.cos(th), r * np.sin(th)], axis=1)
    xy = np.concatenate([core, arms])
    xyz = np.concatenate([xy, rng.normal(0.0, 0.01, (n_stations, 1))], axis=1)
    i, j = np.triu_indices(n_stations, 1)
    bl = torch.tensor(xyz[j] - xyz[i], dtype=torch.float64, device=device)   # (n_bl, 3)
    n_bl = bl.shape[0]
    n_t = -(-n_records // n_bl)
    count = n_records - first if count is None else count
    rec = torch.arange(first, first + count, device=device, dtype=torch.int64)
    tt, bb = rec // n_bl, rec % n_bl
    ha = -math.pi / 3 + (2 * math.pi / 3) * tt.to(torch.float64) / max(n_t - 1, 1)
    dec = math.radians(dec_deg)
    sh, ch = torch.sin(ha), torch.cos(ha)
    bx, by, bz = bl[bb, 0], bl[bb, 1], bl[bb, 2]
    u = sh * bx + ch * by
    v = -math.sin(dec) * ch * bx + math.sin(dec) * sh * by + math.cos(dec) * bz
    w = math.cos(dec) * ch * bx - math.cos(dec) * sh * by + math.sin(dec) * bz
    # global normalisation (identical for every partition)
    bl_len = torch.linalg.norm(bl[:, :2], dim=1).max().item()
    scale = max_uv_frac / bl_len
    wmax = torch.linalg.norm(bl, dim=1).max().item()
    u = 0.5 + u * scale
    v = 0.5 + v * scale
    wn = (w.abs() / wmax).clamp(0.0, 1.0)
    t = (rec * n_time_slices // n_records).to(torch.int32)
    un, vn, wnat = u / cell, v / cell, wn * w_max_native
    val = torch.zeros(count, dtype=torch.complex128, device=device)
    for l, m, f in sources:
        nn = math.sqrt(1.0 - l * l - m * m)
        ph = -2.0 * math.pi * (un * l + vn * m + wnat * (nn - 1.0))
        val += (f / nn) * torch.polar(torch.ones_like(ph), ph)
    vis = val.to(torch.complex64)[:, None].contiguous()
    wt = torch.ones((count, 1), dtype=torch.float32, device=device)
    return u.contiguous(), v.contiguous(), wn.contiguous(), t, vis, wt
