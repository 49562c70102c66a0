"""Multi-slab CUDA stages. (1) R virtual ranks on one GPU, the collectives
replaced by tensor slicing: the slab pipeline must reproduce the single-GPU
image bit for bit. (2) With >= 2 GPUs, the real NCCL driver under
torch.multiprocessing."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, chunk_from, rel_l2

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = Path(__file__).resolve().parents[1]
TESTS = Path(__file__).resolve().parent


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_00959_b200 as W
    return W


def _parts(t, R):
    from oracle import wstack_oracle as O
    sl = np.unique(t)
    out = []
    for r in range(R):
        s0, sc = O.partition_1d(len(sl), R, r)
        out.append((np.searchsorted(t, sl[s0], "left"), np.searchsorted(t, sl[s0 + sc - 1], "right")))
    return out


def _virtual_ranks(W, u, v, w, t, vis, wt, spec, kern, R, n_ranges=1, starts=None):
    from paper_2504_00959_b200.distributed import CudaBackend, norm_sum, plane_ranges
    be = CudaBackend(0)
    G = 1
    S = kern.half_support
    if starts is None:
        slabs = [W.partition_1d(spec.n_v, R, d) for d in range(R)]
    else:
        slabs = [(starts[d], starts[d + 1] - starts[d]) for d in range(R)]
    cols = [W.partition_1d(spec.n_u // G, R, d) for d in range(R)]
    sends = []
    for lo, hi in _parts(t, R):
        rec, pl = be.prepare(u[lo:hi], v[lo:hi], w[lo:hi], vis[lo:hi], wt[lo:hi], spec)
        sends.append(be.route(rec, pl, spec, S, R, starts))
    grids, upd = [], 0
    for d, (v0, vc) in enumerate(slabs):
        recs, pls = [], []
        for srec, spl, counts in sends:            # sources in rank (= gindex) order
            off = sum(counts[:d])
            recs.append(srec[off:off + counts[d]])
            pls.append(spl[off:off + counts[d]])
        gs, up = be.grid_slab(torch.cat(recs).contiguous(), torch.cat(pls).contiguous(), spec, kern,
                              v0, vc)
        grids.append([be.fft_rows(gs, spec, vc, [ng for _, ng in cols], k0, k1)
                      for k0, k1 in plane_ranges(spec.n_w, n_ranges)])
        upd += up
    pix = np.empty((spec.n_v, spec.n_u))
    parts = []
    for d, (g0, ng) in enumerate(cols):
        for i, (k0, k1) in reversed(list(enumerate(plane_ranges(spec.n_w, n_ranges)))):
            # the all-to-all: destination d's block of every source, in source order
            chunks = []
            for (v0, vc), gps in zip(slabs, grids):
                n = (k1 - k0) * vc * G * 2
                start = sum(n * ng_d for _, ng_d in cols[:d])
                chunks.append(gps[i][start:start + n * ng])
            tgrid = torch.cat(chunks).contiguous()
            strip, partials = be.fft_cols_stack(tgrid, spec, [vc for _, vc in slabs], g0, ng, k0, k1)
        pix[:, g0 * G:(g0 + ng) * G] = strip.cpu().numpy()
        parts.append(partials.cpu().numpy().reshape(-1, ng * G, 2))
    p = np.concatenate(parts, axis=1).reshape(-1, 2)   # residue-major, global column order
    return pix, np.sqrt(norm_sum(p)), upd


@pytest.mark.parametrize("R,n_ranges,uneven", [(2, 1, False), (4, 1, False), (8, 1, False),
                                               (2, 3, False), (4, 4, False), (3, 2, True),
                                               (4, 1, True)])
def test_virtual_ranks_bit_identical(W, golden_image, R, n_ranges, uneven):
    g = golden_image
    n_u, n_v, n_w, S, _ = (int(x) for x in g["wide_cfg"])
    cell, wmin, wmax, shape = (float(x) for x in g["wide_fcfg"])
    spec = W.GridSpec(n_u, n_v, n_w, cell, w_min_native=wmin, w_max_native=wmax)
    kern = W.KernelSpec("gaussian", S, shape)
    u, v, w, t, vis, wt = chunk_from(g, "wide_in_")
    ref, diag = W.image(u, v, w, t, vis, wt, spec, kern)
    starts = None
    if uneven:
        # slabs of distinct heights, down to one row (load-balanced slab rows)
        starts = {3: [0, n_v // 5, n_v // 2, n_v], 4: [0, 7, n_v // 2, n_v // 2 + 1, n_v]}[R]
    pix, norms, upd = _virtual_ranks(W, u, v, w, t, vis, wt, spec, kern, R, n_ranges, starts)
    assert upd == diag["grid_updates"]
    assert pix.tobytes() == ref.pixels.tobytes()
    assert norms[0] == ref.imag_residual_norm and norms[1] == ref.real_norm
    assert rel_l2(pix, g["wide_pixels"]) <= 1e-10


def _virtual_plane_ranks(W, u, v, w, t, vis, wt, spec, kern, starts, n_ranges=1):
    """w-plane decomposition with R = len(starts) - 1 virtual ranks on one GPU:
    route by plane, grid + transform + partial stack per rank, the reduce as
    a sum of the partial images, then the finish kernel."""
    import dataclasses
    from paper_2504_00959_b200.distributed import CudaBackend, norm_sum, plane_ranges
    be = CudaBackend(0)
    R = len(starts) - 1
    sends = []
    for lo, hi in _parts(t, R):
        rec, pl = be.prepare(u[lo:hi], v[lo:hi], w[lo:hi], vis[lo:hi], wt[lo:hi], spec)
        assert int(be.plane_histogram(pl, spec).sum()) == hi - lo
        sends.append(be.route_planes(rec, pl, spec, R, starts))
    total = None
    upd = 0
    for d in range(R):
        recs, pls = [], []
        for srec, spl, counts in sends:
            off = sum(counts[:d])
            recs.append(srec[off:off + counts[d]])
            pls.append(spl[off:off + counts[d]])
        p0, p1 = starts[d], starts[d + 1]
        spec_l = dataclasses.replace(spec, n_w=p1 - p0)
        gs, up = be.grid_slab(torch.cat(recs).contiguous(), torch.cat(pls).contiguous(), spec_l,
                              kern, 0, spec.n_v)
        upd += up
        pimg = torch.empty((spec.n_v, spec.n_u, 2), dtype=torch.float64, device=be.device)
        for l0, l1 in reversed(plane_ranges(p1 - p0, n_ranges)):
            gp = be.fft_rows(gs, spec_l, spec.n_v, [spec.n_u], l0, l1)
            be.fft_cols_partial(gp, spec, p0 + l0, p0 + l1, p0, p1, pimg)
        total = pimg if total is None else total + pimg
    pix, parts = be.image_finish(total, spec)
    p = parts.reshape(-1, 2).cpu().numpy()
    return pix.cpu().numpy(), np.sqrt(norm_sum(p)), upd


@pytest.mark.parametrize("starts,n_ranges", [([0, 8, 16], 1), ([0, 3, 9, 10, 16], 1),
                                             ([0, 5, 16], 3), ([0, 16], 2)])
def test_virtual_plane_ranks(W, golden_image, starts, n_ranges):
    g = golden_image
    n_u, n_v, n_w, S, _ = (int(x) for x in g["wide_cfg"])
    cell, wmin, wmax, shape = (float(x) for x in g["wide_fcfg"])
    spec = W.GridSpec(n_u, n_v, n_w, cell, w_min_native=wmin, w_max_native=wmax)
    kern = W.KernelSpec("gaussian", S, shape)
    u, v, w, t, vis, wt = chunk_from(g, "wide_in_")
    ref, diag = W.image(u, v, w, t, vis, wt, spec, kern)
    pix, norms, upd = _virtual_plane_ranks(W, u, v, w, t, vis, wt, spec, kern, starts, n_ranges)
    assert upd == diag["grid_updates"]
    assert rel_l2(pix, ref.pixels) <= 1e-13
    np.testing.assert_allclose(norms, [ref.imag_residual_norm, ref.real_norm], rtol=1e-12)
    assert rel_l2(pix, g["wide_pixels"]) <= 1e-10


def test_virtual_plane_ranks_split_transforms(W):
    """8192^2 mesh (split row/column transforms, SP = 2) through the partial
    stack: equals the single-GPU image to rounding."""
    rng = np.random.default_rng(11)
    n = 200_000
    spec = W.GridSpec(8192, 8192, 4, 2e-5, w_max_native=300.0)
    kern = W.KernelSpec.gaussian(2, 1.0)
    u, v = rng.uniform(0.3, 0.7, n), rng.uniform(0.3, 0.7, n)
    w = rng.uniform(0.0, 1.0, n)
    t = np.sort(rng.integers(0, 64, n))
    vis = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
    wt = rng.uniform(0.5, 1.0, n).astype(np.float32)
    ref, diag = W.image(u, v, w, t, vis, wt, spec, kern)
    pix, norms, upd = _virtual_plane_ranks(W, u, v, w, t, vis, wt, spec, kern, [0, 1, 4])
    assert upd == diag["grid_updates"]
    assert rel_l2(pix, ref.pixels) <= 1e-13
    np.testing.assert_allclose(norms, [ref.imag_residual_norm, ref.real_norm], rtol=1e-12)


@pytest.mark.parametrize("R", [2, 4])
def test_virtual_ranks_bit_identical_with_split_items(W, R):
    """Dense uv coverage (Earth-rotation-like clustering) puts more than one
    work part's worth of records into single gridder items, which are then
    gridded in parts and combined in part order. With slabs on the 128-row
    item boundaries (partition_1d of 512 rows over 2/4 ranks) every item
    holds the same records as on one GPU: the v-slab image stays bit-identical."""
    rng = np.random.default_rng(23)
    n = 400_000
    u = np.clip(rng.normal(0.5, 0.01, n), 0, 1 - 1e-9)
    v = np.clip(rng.normal(0.5, 0.01, n), 0, 1 - 1e-9)
    w = rng.uniform(0.0, 1.0, n)
    t = np.sort(rng.integers(0, 16, n)).astype(np.uint32)
    vis = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
    wt = rng.uniform(0.5, 1.0, n).astype(np.float32)
    spec = W.GridSpec(512, 512, 4, 2e-4, w_max_native=200.0)
    kern = W.KernelSpec.gaussian(3, 1.0)
    ref, diag = W.image(u, v, w, t, vis, wt, spec, kern)
    pix, norms, upd = _virtual_ranks(W, u, v, w, t, vis, wt, spec, kern, R)
    assert upd == diag["grid_updates"]
    assert pix.tobytes() == ref.pixels.tobytes()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl_worker(rank, world, port, outdir):
    sys.path[:0] = [str(ROOT), str(TESTS)]
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        import paper_2504_00959_b200 as W
        from paper_2504_00959_b200.distributed import image_distributed
        g = np.load(TESTS / "golden" / "image.npz")
        n_u, n_v, n_w, S, _ = (int(x) for x in g["wide_cfg"])
        cell, wmin, wmax, shape = (float(x) for x in g["wide_fcfg"])
        spec = W.GridSpec(n_u, n_v, n_w, cell, w_min_native=wmin, w_max_native=wmax)
        kern = W.KernelSpec("gaussian", S, shape)
        u, v, w, t, vis, wt = (g[f"wide_in_{k}"] for k in ("u", "v", "w", "time_index", "vis", "weight"))
        lo, hi = _parts(t, world)[rank]
        dev = torch.device("cuda", rank)
        args = [torch.from_numpy(np.ascontiguousarray(a[lo:hi])).to(dev) for a in (u, v, w, vis, wt)]
        outs = {}
        # fused peer-memory transpose (twice: the symmetric buffer is reused),
        # the pipelined NCCL all-to-all, and partition_1d slabs
        sl = dict(decomposition="slabs")
        for name, kw in (("push", dict(transpose="push", **sl)), ("push2", dict(transpose="push", **sl)),
                         ("peer", dict(transpose="peer", **sl)),
                         ("nccl", dict(transpose="nccl", **sl)),
                         ("xnccl", dict(exchange="nccl", transpose="nccl", **sl)),
                         ("even", dict(transpose="nccl", balance=False, **sl)),
                         ("planes", dict(decomposition="planes")),
                         ("planes_even", dict(decomposition="planes", balance=False)),
                         ("planes_xnccl", dict(decomposition="planes", exchange="nccl"))):
            img, diag = image_distributed(*args, spec, kern, **kw)
            if rank == 0:
                outs[name] = img.pixels
                outs[name + "_updates"] = np.array([diag["grid_updates"]])
                outs[name + "_norms"] = np.array([img.imag_residual_norm, img.real_norm])
        # the double-buffered stream API: this rank's slice in two batches
        from paper_2504_00959_b200.distributed import image_distributed_stream
        mid = (lo + hi) // 2
        batches = [tuple(np.ascontiguousarray(x[a_:b_]) for x in (u, v, w, vis, wt))
                   for a_, b_ in ((lo, mid), (mid, hi))]
        for bi, (img, diag) in enumerate(image_distributed_stream(batches, spec, kern,
                                                                  decomposition="slabs")):
            if rank == 0:
                outs[f"stream{bi}"] = img.pixels
        for bi, (img, diag) in enumerate(image_distributed_stream(batches, spec, kern)):  # auto
            if rank == 0:
                outs[f"pstream{bi}"] = img.pixels
        # multi-GPU ingest: every rank reads its own time partition of an RVIS
        # dataset (run_pipeline over the process group)
        from paper_2504_00959_b200.distributed import run_pipeline_distributed
        res = run_pipeline_distributed(TESTS / "golden" / "chunks.rvis", 64, 64, 4, 1e-3,
                                       W.KernelSpec.gaussian(3, 1.0), out_dir=Path(outdir) / "rpd")
        if rank == 0:
            outs["rpd_pixels"] = res.image.pixels
            outs["rpd_ops"] = np.array([res.ops[k] for k in _OPS])
            outs["rpd_phases"] = np.array(sorted(res.run.phase_times))
        else:
            assert res is None
        if rank == 0:
            np.savez(Path(outdir) / "out.npz", **outs)
    finally:
        dist.destroy_process_group()


_OPS = ("records", "grid_updates", "exchange_bytes", "reduce_bytes", "fft_bytes",
        "reduce_messages", "stack_pixels")


class _Topo:
    def __init__(self, n_nodes, ranks_per_node):
        self.n_nodes, self.ranks_per_node, self.threads_per_rank = n_nodes, ranks_per_node, 1
        self.n_ranks = n_nodes * ranks_per_node


def test_nccl_multi_gpu_matches_single(W, golden_image, tmp_path):
    world = min(torch.cuda.device_count(), 4)
    if world < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp
    mp.spawn(_nccl_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    out = np.load(tmp_path / "out.npz")
    g = golden_image
    n_u, n_v, n_w, S, _ = (int(x) for x in g["wide_cfg"])
    cell, wmin, wmax, shape = (float(x) for x in g["wide_fcfg"])
    spec = W.GridSpec(n_u, n_v, n_w, cell, w_min_native=wmin, w_max_native=wmax)
    ref, diag = W.image(*chunk_from(g, "wide_in_"), spec, W.KernelSpec("gaussian", S, shape))
    for name in ("push", "push2", "peer", "nccl", "xnccl", "even"):
        assert int(out[name + "_updates"][0]) == diag["grid_updates"], name
        assert out[name].tobytes() == ref.pixels.tobytes(), name
    # w-plane decomposition: the stack's association over planes depends on
    # the ranks -- equal to rounding, not bitwise
    for name in ("planes", "planes_even", "planes_xnccl"):
        assert int(out[name + "_updates"][0]) == diag["grid_updates"], name
        err = np.linalg.norm(out[name] - ref.pixels) / np.linalg.norm(ref.pixels)
        assert err <= 1e-13, (name, err)
        np.testing.assert_allclose(out[name + "_norms"], [ref.imag_residual_norm, ref.real_norm],
                                   rtol=1e-12)
        err_g = np.linalg.norm(out[name] - g["wide_pixels"]) / np.linalg.norm(g["wide_pixels"])
        assert err_g <= 1e-10, (name, err_g)
    # stream batches: batch b = every rank's b-th half of its slice, in rank order
    u, v, w, t, vis, wt = chunk_from(g, "wide_in_")
    parts = _parts(t, world)
    for bi in range(2):
        sel = np.concatenate([np.arange(lo, (lo + hi) // 2) if bi == 0 else np.arange((lo + hi) // 2, hi)
                              for lo, hi in parts])
        ref_b, _ = W.image(*(x[sel] for x in (u, v, w)), None, vis[sel], wt[sel], spec,
                           W.KernelSpec("gaussian", S, shape))
        assert out[f"stream{bi}"].tobytes() == ref_b.pixels.tobytes(), bi
        err = np.linalg.norm(out[f"pstream{bi}"] - ref_b.pixels) / np.linalg.norm(ref_b.pixels)
        assert err <= 1e-13, (bi, err)
    # run_pipeline_distributed vs the single-GPU run_pipeline on topology 1 x world
    one = W.run_pipeline(GOLDEN / "chunks.rvis", 64, 64, 4, 1e-3, W.KernelSpec.gaussian(3, 1.0),
                         topo=_Topo(1, world), out_dir=tmp_path / "one")
    err = np.linalg.norm(out["rpd_pixels"] - one.image.pixels) / np.linalg.norm(one.image.pixels)
    assert err <= 1e-13, err
    assert [int(x) for x in out["rpd_ops"]] == [one.ops[k] for k in _OPS]
    assert (tmp_path / "rpd" / "messages.csv").read_text() == (tmp_path / "one" / "messages.csv").read_text()
    assert list(out["rpd_phases"]) == ["fft", "gridding", "read", "reduce", "total", "wcorrect", "write"]
