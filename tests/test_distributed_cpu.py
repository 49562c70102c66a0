"""Multi-rank host logic of distributed.image_distributed on CPU: gloo,
world_size 2 and 4, stage math from the oracle-backed NumpyBackend. Checks the
exchange splits, per-plane transposes and the image/norm gathers against the
single-process oracle image."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
TESTS = Path(__file__).resolve().parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, outdir, row_weight, decomp="slabs"):
    sys.path[:0] = [str(ROOT), str(TESTS)]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from np_backend import NumpyBackend
        from oracle import wstack_oracle as O
        import paper_2504_00959_b200 as W
        from paper_2504_00959_b200.distributed import image_distributed

        g = np.load(TESTS / "golden" / "image.npz")
        n_u, n_v, n_w, S, _ = (int(x) for x in g[f"{case}_cfg"])
        cell, wmin, wmax, shape = (float(x) for x in g[f"{case}_fcfg"])
        kind = "gaussian" if int(g[f"{case}_kind"][0]) == 0 else "kaiser_bessel"
        u, v, w, t = (g[f"{case}_in_{k}"] for k in ("u", "v", "w", "time_index"))
        vis, wt = g[f"{case}_in_vis"], g[f"{case}_in_weight"]
        # time-ordered partition (visdata.py:344-366)
        sl = np.unique(t)
        s0, sc = O.partition_1d(len(sl), world, rank)
        lo = np.searchsorted(t, sl[s0], "left")
        hi = np.searchsorted(t, sl[s0 + sc - 1], "right")
        spec = W.GridSpec(n_u, n_v, n_w, cell, w_min_native=wmin, w_max_native=wmax)
        kern = W.KernelSpec(kind, S, shape)
        img, diag = image_distributed(u[lo:hi], v[lo:hi], w[lo:hi], vis[lo:hi], wt[lo:hi], spec,
                                      kern, backend=NumpyBackend(), row_weight=row_weight,
                                      decomposition=decomp)
        if rank == 0:
            starts = diag["slab_starts"] if decomp == "slabs" else diag["plane_starts"]
            np.savez(Path(outdir) / "out.npz", pixels=img.pixels, starts=np.array(starts),
                     norms=np.array([img.imag_residual_norm, img.real_norm]),
                     updates=np.array([diag["grid_updates"]]))
    finally:
        dist.destroy_process_group()


# row_weight 1.0: slabs sized by the records alone (uneven rows); 1e9: the
# equal-row partition
@pytest.mark.parametrize("world,case,row_weight", [(2, "wide", 1e9), (4, "wide", 1e9),
                                                   (2, "kb1", 1e9), (2, "wide", 1.0),
                                                   (4, "wide", 1.0)])
def test_image_distributed_gloo(tmp_path, golden_image, world, case, row_weight):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, case, str(tmp_path), row_weight), nprocs=world, join=True)
    out = np.load(tmp_path / "out.npz")
    starts = out["starts"]
    assert starts[0] == 0 and starts[-1] == golden_image[f"{case}_cfg"][1] and np.all(np.diff(starts) > 0)
    g = golden_image
    ref = g[f"{case}_pixels"]
    err = float(np.linalg.norm(out["pixels"] - ref) / np.linalg.norm(ref))
    assert err <= 1e-12, err
    assert int(out["updates"][0]) == int(g[f"{case}_grid_updates"][0])
    np.testing.assert_allclose(out["norms"], g[f"{case}_norms"], rtol=1e-10)


# w-plane decomposition: plane ranges, partial stacks summed on the root;
# row_weight is unused there (plane_weight default)
@pytest.mark.parametrize("world,case", [(2, "wide"), (4, "wide"), (2, "kb1"), (4, "small")])
def test_image_distributed_planes_gloo(tmp_path, golden_image, world, case):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, case, str(tmp_path), 1.0, "planes"), nprocs=world,
             join=True)
    out = np.load(tmp_path / "out.npz")
    starts = out["starts"]
    g = golden_image
    assert starts[0] == 0 and starts[-1] == g[f"{case}_cfg"][2] and np.all(np.diff(starts) > 0)
    assert len(starts) == world + 1
    ref = g[f"{case}_pixels"]
    err = float(np.linalg.norm(out["pixels"] - ref) / np.linalg.norm(ref))
    assert err <= 1e-12, err
    assert int(out["updates"][0]) == int(g[f"{case}_grid_updates"][0])
    np.testing.assert_allclose(out["norms"], g[f"{case}_norms"], rtol=1e-10)


def test_balanced_slab_starts():
    from paper_2504_00959_b200.distributed import balanced_slab_starts
    h = np.zeros(64, np.int64)
    h[28:36] = 1000                       # records piled in the central rows
    st = balanced_slab_starts(h, 4, row_weight=0.0, max_rows=64)
    assert st[0] == 0 and st[-1] == 64 and all(b > a for a, b in zip(st, st[1:]))
    # the central block is cut into four (nearly) equal parts
    per = [h[a:b].sum() for a, b in zip(st, st[1:])]
    assert max(per) - min(per) <= 1000
    # huge row weight -> equal rows
    assert balanced_slab_starts(h, 4, row_weight=1e12) == [0, 16, 32, 48, 64]
    # more ranks than loaded rows still gives non-empty slabs
    st = balanced_slab_starts(np.eye(1, 8, 7, dtype=np.int64)[0] * 10, 8, row_weight=0.0)
    assert st == list(range(9))
    # the memory cap: no slab above 1.5x the equal share by default
    st = balanced_slab_starts(h, 4, row_weight=0.0)
    assert max(b - a for a, b in zip(st, st[1:])) <= 24 and st[-1] == 64


def test_balanced_slab_starts_align_to_gridder_items():
    """Balanced slabs start on the gridder's 128-row item boundaries (the
    condition for a bit-identical image across GPU counts) when the mesh has
    room for it; memory caps and the ordering still hold."""
    from paper_2504_00959_b200.distributed import ITEM_ROWS, balanced_slab_starts
    rng = np.random.default_rng(3)
    h = rng.poisson(5, 2048)
    h[900:1100] += 5000                    # dense central rows
    for R in (2, 3, 4, 8):
        st = balanced_slab_starts(h, R, row_weight=100.0)
        assert st[0] == 0 and st[-1] == 2048 and all(b > a for a, b in zip(st, st[1:]))
        assert all(s % ITEM_ROWS == 0 for s in st), (R, st)
    # no room (fewer than 128 rows per rank): unaligned but valid
    st = balanced_slab_starts(h[:512], 8, row_weight=1.0)
    assert st[0] == 0 and st[-1] == 512 and all(b > a for a, b in zip(st, st[1:]))
