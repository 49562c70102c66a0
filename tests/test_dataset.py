"""RVIS ingest: the reader against the reference's own
reads of a reference-written file (whole file, a time chunk, a frequency
chunk), the writer round trip, the chunk rules, and (GPU) streamed imaging
of time chunks."""

from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def W():
    import paper_2504_00959_b200 as W
    return W


def _same(cols, g, tag):
    for k in ("u", "v", "w", "time_index", "vis", "weight"):
        a, b = np.asarray(cols[k]), g[f"{tag}_{k}"]
        assert a.shape == b.shape and a.dtype == b.dtype, (k, a.shape, b.shape, a.dtype, b.dtype)
        assert a.tobytes() == b.tobytes(), k


@pytest.mark.parametrize("tag,spec", [("all", None), ("t1of3", ("time", 1, 3)),
                                      ("f1of3", ("frequency", 1, 3))])
def test_read_dataset_matches_reference(W, tag, spec):
    g = np.load(GOLD / "rvis.npz")
    chunk = None if spec is None else W.ChunkSpec(*spec)
    header, cols = W.read_dataset(GOLD / "chunks.rvis", chunk)
    assert header["n_freq"] == 3 and header["n_corr"] == 2 and header["n_time_slices"] == 8
    assert header["reserved"][:5] == b"pcg64"     # generator provenance kept
    _same(cols, g, tag)


def test_time_chunks_cover_once_and_roundtrip(W, tmp_path):
    header, cols = W.read_dataset(GOLD / "chunks.rvis")
    idx = []
    for i in range(3):
        _, c = W.read_dataset(GOLD / "chunks.rvis", W.ChunkSpec("time", i, 3))
        idx.append(c["u"])
    assert np.array_equal(np.concatenate(idx), cols["u"])     # time-sorted file: chunks in order
    p = tmp_path / "copy.rvis"
    W.write_dataset(cols, header, p)
    assert p.read_bytes() == (GOLD / "chunks.rvis").read_bytes()
    with pytest.raises(ValueError):
        W.ChunkSpec("space", 0, 1)
    with pytest.raises(ValueError):
        W.ChunkSpec("time", 3, 3)


def test_truncated_file_rejected(W, tmp_path):
    raw = (GOLD / "chunks.rvis").read_bytes()
    p = tmp_path / "short.rvis"
    p.write_bytes(raw[:-5])
    with pytest.raises(W.FormatError):
        W.read_dataset(p)


@pytest.mark.gpu
def test_image_time_chunks_streamed(W):
    header, _ = W.read_dataset(GOLD / "chunks.rvis")
    spec = W.GridSpec(64, 64, 4, 1e-3, w_min_native=header["w_min_native"],
                      w_max_native=header["w_max_native"])
    kern = W.KernelSpec.gaussian(3, 1.0)
    got = list(W.image_time_chunks(GOLD / "chunks.rvis", spec, kern, 3))
    assert len(got) == 3
    for i, (img, diag) in enumerate(got):
        _, c = W.read_dataset(GOLD / "chunks.rvis", W.ChunkSpec("time", i, 3))
        ref, dref = W.image(c["u"], c["v"], c["w"], None, c["vis"], c["weight"], spec, kern)
        assert img.pixels.tobytes() == ref.pixels.tobytes()
        assert diag["grid_updates"] == dref["grid_updates"]


@pytest.mark.parametrize("R", [1, 2, 3, 4, 8])
def test_rank_partitions_read_only_their_rows(W, R):
    """Multi-GPU ingest (run_pipeline_distributed): rank r reads records
    [lo, hi) of the r-th time partition (_partition_for_ranks,
    pipeline.py:47-58); the partitions tile the file in order."""
    from paper_2504_00959_b200.imager import _partition_bounds
    _, cols = W.read_dataset(GOLD / "chunks.rvis")
    bounds, ordered = _partition_bounds(cols["time_index"], R)
    assert ordered and bounds[0][0] == 0 and bounds[-1][1] == len(cols["u"])
    assert all(a[1] == b[0] for a, b in zip(bounds, bounds[1:]))
    for lo, hi in bounds:
        _, part = W.read_dataset(GOLD / "chunks.rvis", rows=(lo, hi))
        for k in ("u", "v", "w", "time_index", "vis", "weight"):
            assert part[k].tobytes() == cols[k][lo:hi].tobytes(), k
        # a partition holds whole time slices
        if hi < len(cols["u"]):
            assert cols["time_index"][hi - 1] != cols["time_index"][hi]
