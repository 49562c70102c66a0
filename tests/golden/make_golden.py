"""Generate golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference ``wstack`` package read-only from
``/root/reference/pkg/src`` and stores its outputs (bucketing batches,
grids, images) plus the inputs that produced them as small ``.npz`` files
next to this script. The fixtures travel with the repo; nothing at test time
reads ``/root/reference``.
"""

from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import wstack  # noqa: F401
    from wstack import comms, gridder, mesh, pipeline, visdata
    return comms, gridder, mesh, pipeline, visdata


def edge_case_chunk(visdata, n_u, n_v, n_w, n_chan=1, seed=3):
    """Hand-placed records on every boundary the bucketing rules have."""
    rng = np.random.default_rng(seed)
    tiny = np.nextafter(0.0, 1.0)
    below1 = np.nextafter(1.0, 0.0)
    u, v, w = [], [], []
    # corners / edges of the uv square
    for uu in (0.0, tiny, 0.5, below1, 1.0 / n_u, 3.0 / n_u, 1.0 - 3.0 / n_u):
        for vv in (0.0, tiny, below1, 0.5, 2.0 / n_v, 1.0 - 2.5 / n_v):
            u.append(uu)
            v.append(vv)
            w.append(rng.random())
    # exact integer cells, exact half cells
    for k in range(12):
        u.append((7 + k) / n_u)
        v.append((9 + 2 * k) / n_v)
        w.append(rng.random())
        u.append((7.5 + k) / n_u)
        v.append((9.5 + k) / n_v)
        w.append(rng.random())
    # rows straddling the slab boundaries of 2/4/8 slabs, +-S around them
    for r in (2, 4, 8):
        for b in range(1, r):
            vb = b * n_v // r
            for off in (-3.5, -3.0, -2.999, -0.5, 0.0, 0.25, 2.0, 3.0, 3.0001):
                vv = (vb + off) / n_v
                if 0.0 <= vv < 1.0:
                    u.append(rng.random())
                    v.append(vv)
                    w.append(rng.random())
    # w exactly on plane boundaries and ends
    for k in range(n_w):
        for ww in ((k + 0.5) / max(n_w - 1, 1), k / max(n_w - 1, 1),
                   np.nextafter((k + 0.5) / max(n_w - 1, 1), 0.0)):
            if 0.0 <= ww <= 1.0:
                u.append(rng.random())
                v.append(rng.random())
                w.append(ww)
    w.extend([0.0, 1.0])
    u.extend([0.25, 0.75])
    v.extend([0.25, 0.75])
    n = len(u)
    vis = (rng.standard_normal((n, n_chan)) + 1j * rng.standard_normal((n, n_chan))).astype(np.complex64)
    weight = rng.random((n, n_chan)).astype(np.float32)
    weight[::5] = 0.0
    t = np.sort(rng.integers(0, 8, n)).astype(np.uint32)
    return visdata.VisChunk(np.array(u), np.array(v), np.array(w), t, vis, weight)


def chunk_arrays(prefix, chunk):
    return {f"{prefix}u": chunk.u, f"{prefix}v": chunk.v, f"{prefix}w": chunk.w,
            f"{prefix}time_index": chunk.time_index, f"{prefix}vis": chunk.vis,
            f"{prefix}weight": chunk.weight}


def make_bucket(comms, gridder, mesh, visdata):
    """exchange_to_space_order batches at 1/2/4/8 ranks (comms.py:495-547)."""
    out = {}
    sky = visdata.SkyModel(sources=((0.01, -0.008, 2.0), (0.0, 0.0, 1.0)))
    _, chunk = visdata.generate_synthetic(sky, 1000, 2, seed=11, n_time_slices=8,
                                          cell_size_lm=1e-3, w_min_native=0.0,
                                          w_max_native=12.0)
    cases = {"syn": (chunk, 64, 64, 4, 3), "edge": (edge_case_chunk(visdata, 64, 64, 5), 64, 64, 5, 3)}
    for name, (ch, n_u, n_v, n_w, S) in cases.items():
        out.update(chunk_arrays(f"{name}_in_", ch))
        out[f"{name}_spec"] = np.array([n_u, n_v, n_w, S])
        spec = mesh.GridSpec(n_u=n_u, n_v=n_v, n_w=n_w, cell_size_lm=1e-3)
        prep = comms.prepare_chunk(ch, spec, 0)
        for k in ("gu", "gv", "plane", "value", "gindex"):
            out[f"{name}_prep_{k}"] = prep[k]
        for R in (1, 2, 4, 8):
            topo = comms.Topology(1, R)
            parts = visdata.partition_time_ordered(ch, R)
            batches = comms.exchange_to_space_order(parts, spec, topo, halo_rows=S)
            for d, b in enumerate(batches):
                key = f"{name}_R{R}_d{d}_"
                for col in ("gu", "gv", "plane", "value", "time_index", "gindex", "is_halo"):
                    out[key + col] = getattr(b, col)
    np.savez_compressed(HERE / "bucket.npz", **out)


def make_grid(comms, gridder, mesh, visdata):
    """grid_all gathered slabs + grid_updates (gridder.py:262-294)."""
    out = {}
    sky = visdata.SkyModel(sources=((0.01, -0.008, 2.0), (0.0, 0.0, 1.0)))
    _, chunk = visdata.generate_synthetic(sky, 1000, 2, seed=11, n_time_slices=8,
                                          cell_size_lm=1e-3, w_min_native=0.0,
                                          w_max_native=12.0)
    out.update(chunk_arrays("in_", chunk))
    spec = mesh.GridSpec(n_u=64, n_v=64, n_w=4, cell_size_lm=1e-3,
                         w_min_native=0.0, w_max_native=12.0)
    kernels = {
        "gauss3": gridder.KernelSpec.gaussian(3, 1.0),
        "gauss1": gridder.KernelSpec.gaussian(1, 0.7),
        "kb1": gridder.KernelSpec.kaiser_bessel(1),
        "kb3": gridder.KernelSpec.kaiser_bessel(3),
        "kb5": gridder.KernelSpec.kaiser_bessel(5),
    }
    for name, kern in kernels.items():
        for R in (1, 2, 4):
            topo = comms.Topology(1, R)
            parts = visdata.partition_time_ordered(chunk, R)
            slabs, _ = gridder.grid_all(parts, spec, kern, topo)
            g = np.concatenate([s.data for s in slabs], axis=1)
            if R == 1:
                out[f"{name}_grid"] = g
                out[f"{name}_shape"] = np.array([kern.shape_param])
                out[f"{name}_S"] = np.array([kern.half_support])
            else:
                assert g.tobytes() == out[f"{name}_grid"].tobytes()
        # update count for one rank (grid_sector return value)
        batches = comms.exchange_to_space_order([chunk], spec, comms.Topology(1, 1),
                                                halo_rows=kern.half_support)
        cg = mesh.ComplexGrid(spec, mesh.slab_of(spec, 0, 1))
        out[f"{name}_updates"] = np.array([gridder.grid_sector(batches[0], kern, cg)])
    np.savez_compressed(HERE / "grid.npz", **out)


def make_images(comms, gridder, mesh, pipeline, visdata):
    """run_pipeline images (pipeline.py:61-191) for several configurations."""
    out = {}
    rng_sources = ((0.02, -0.015, 2.0), (0.0, 0.0, 1.0))
    cases = [
        # name, n_u, n_v, n_w, cell, wmax, n_rec, n_freq, kernel, seed, ranks
        ("small", 64, 64, 4, 1e-3, 20.0, 1000, 2, gridder.KernelSpec.gaussian(3, 1.0), 90, 2),
        ("kb5", 128, 128, 8, 1e-3, 50.0, 4000, 1, gridder.KernelSpec.kaiser_bessel(5), 5, 1),
        ("kb1", 64, 32, 3, 2e-3, 30.0, 1500, 1, gridder.KernelSpec.kaiser_bessel(1), 6, 2),
        ("nw1", 32, 32, 1, 1e-3, 10.0, 500, 1, gridder.KernelSpec.gaussian(2, 1.3), 7, 1),
        ("wide", 256, 128, 16, 5e-4, 800.0, 20000, 1, gridder.KernelSpec.gaussian(3, 1.0), 8, 4),
        ("multichan", 64, 64, 6, 1e-3, 100.0, 2000, 7, gridder.KernelSpec.gaussian(3, 0.8), 9, 1),
    ]
    for name, n_u, n_v, n_w, cell, wmax, n_rec, n_freq, kern, seed, ranks in cases:
        sky = visdata.SkyModel(sources=rng_sources)
        header, chunk = visdata.generate_synthetic(
            sky, n_rec, n_freq, seed=seed, n_time_slices=8, cell_size_lm=cell,
            w_min_native=0.0, w_max_native=wmax)
        if name == "multichan":
            # distinct per-channel values and weights exercise the channel sum
            rng = np.random.default_rng(seed)
            chunk = visdata.VisChunk(
                chunk.u, chunk.v, chunk.w, chunk.time_index,
                (chunk.vis * (1 + 0.1 * rng.standard_normal(chunk.vis.shape))).astype(np.complex64),
                rng.random(chunk.weight.shape).astype(np.float32))
        with tempfile.TemporaryDirectory() as tmp:
            path = Path(tmp) / "d.rvis"
            visdata.write_dataset(chunk, header, path)
            res = pipeline.run_pipeline(path, n_u, n_v, n_w, cell, kernel=kern,
                                        topo=comms.Topology(1, ranks), label=name)
        p = f"{name}_"
        out.update(chunk_arrays(p + "in_", chunk))
        out[p + "cfg"] = np.array([n_u, n_v, n_w, kern.half_support, ranks])
        out[p + "fcfg"] = np.array([cell, header.w_min_native, header.w_max_native, kern.shape_param])
        out[p + "kind"] = np.array([0 if kern.kind == "gaussian" else 1])
        out[p + "pixels"] = res.image.pixels
        out[p + "norms"] = np.array([res.image.imag_residual_norm, res.image.real_norm])
        out[p + "grid_updates"] = np.array([res.ops["grid_updates"]])
    np.savez_compressed(HERE / "image.npz", **out)


def make_rvis(visdata):
    """A small multi-channel RVIS file written by the reference and the
    reference's own reads of it: whole, time chunk 1 of 3, frequency chunk 1
    of 3 (visdata.py:312-341)."""
    sky = visdata.SkyModel(sources=((0.01, -0.008, 2.0), (0.0, 0.0, 1.0)))
    header, chunk = visdata.generate_synthetic(sky, 1500, 3, seed=13, n_corr=2, n_time_slices=8,
                                               cell_size_lm=1e-3, w_min_native=0.0,
                                               w_max_native=40.0)
    path = HERE / "chunks.rvis"
    visdata.write_dataset(chunk, header, path)
    out = {}
    for tag, spec in (("all", None), ("t1of3", visdata.ChunkSpec("time", 1, 3)),
                      ("f1of3", visdata.ChunkSpec("frequency", 1, 3))):
        _, c = visdata.read_dataset(path, spec)
        out.update(chunk_arrays(tag + "_", c))
    np.savez_compressed(HERE / "rvis.npz", **out)


PIPELINE_CASES = [
    # name, n_nodes, ranks_per_node, reduce kind, deterministic
    ("t1x1", 1, 1, "direct", True),
    ("t1x3", 1, 3, "direct", True),
    ("t2x2h", 2, 2, "hybrid_ring", True),
    ("t2x3r", 2, 3, "ring_rdma_like", True),
    ("t3x2d", 3, 2, "direct", False),
    ("t1x4h", 1, 4, "hybrid_ring", True),
    ("t2x2r", 2, 2, "ring_rdma_like", False),
]


def make_pipeline(comms, metrics, pipeline):
    """run_pipeline (pipeline.py:61-191) on chunks.rvis for several virtual
    topologies and reduce strategies with a SyntheticPowerMeter: the written
    messages.csv, the ops totals, the per-phase energy keys and the image."""
    out = {}
    path = HERE / "chunks.rvis"
    kern = __import__("wstack.gridder", fromlist=["KernelSpec"]).KernelSpec.gaussian(3, 1.0)
    for name, nn, rpn, kind, det in PIPELINE_CASES:
        with tempfile.TemporaryDirectory() as tmp:
            res = pipeline.run_pipeline(path, 64, 64, 4, 1e-3, kernel=kern,
                                        topo=comms.Topology(nn, rpn),
                                        strategy=comms.ReduceStrategy(kind, det),
                                        meter=metrics.SyntheticPowerMeter(), freq_level="medium",
                                        label=name, out_dir=tmp)
            csv_text = Path(res.paths["messages"]).read_text()
        p = f"{name}_"
        out[p + "topo"] = np.array([nn, rpn, int(det)])
        out[p + "kind"] = np.array(kind)
        out[p + "messages_csv"] = np.array(csv_text)
        out[p + "ops"] = np.array([res.ops[k] for k in ("records", "grid_updates", "exchange_bytes",
                                                          "reduce_bytes", "fft_bytes",
                                                          "reduce_messages", "stack_pixels")])
        out[p + "energy_keys"] = np.array(sorted(res.run.energy_joules))
        out[p + "pixels"] = res.image.pixels
    np.savez_compressed(HERE / "pipeline.npz", **out)


def main():
    comms, gridder, mesh, pipeline, visdata = _ref()
    if sys.argv[1:] == ["rvis"]:
        make_rvis(visdata)
        return
    from wstack import metrics
    if sys.argv[1:] == ["pipeline"]:
        make_pipeline(comms, metrics, pipeline)
        return
    make_bucket(comms, gridder, mesh, visdata)
    make_grid(comms, gridder, mesh, visdata)
    make_images(comms, gridder, mesh, pipeline, visdata)
    make_rvis(visdata)
    make_pipeline(comms, metrics, pipeline)
    for f in sorted(HERE.glob("*.npz")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
