"""The reference's own gridder and pipeline tests, replayed against the GPU
drop-in (paper_2504_00959_b200.grid_sector / grid_all / run_pipeline).

Sector tests restate /root/reference/pkg/tests/test_gridder.py:117-280 with
the same inputs and tolerances; expected values come from the closed forms
those tests use or from the pinned CPU oracle. The run_pipeline tests
compare with tests/golden/pipeline.npz, written by the reference's own
run_pipeline on tests/golden/chunks.rvis for several virtual topologies and
reduce strategies (make_golden.py). Needs a B200."""

import math

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2
from oracle import wstack_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_00959_b200 as W
    return W


class Topo:
    """The fields of the reference's Topology (comms.py:67-97)."""

    def __init__(self, n_nodes, ranks_per_node, threads_per_rank=1):
        self.n_nodes, self.ranks_per_node = n_nodes, ranks_per_node
        self.threads_per_rank = threads_per_rank

    @property
    def n_ranks(self):
        return self.n_nodes * self.ranks_per_node


class Strategy:
    def __init__(self, kind="direct", deterministic=True):
        self.kind, self.deterministic = kind, deterministic


class Chunk:
    def __init__(self, u, v, w, t, vis, wt):
        self.u, self.v, self.w, self.time_index, self.vis, self.weight = u, v, w, t, vis, wt

    def rows(self, sl):
        return Chunk(*(a[sl] for a in (self.u, self.v, self.w, self.time_index, self.vis,
                                       self.weight)))


def _batch(W, spec, slab, gu, gv, plane, value, halo=3):
    return W.SectorBatch(slab, np.asarray(gu, float), np.asarray(gv, float),
                         np.asarray(plane, np.uint32), np.asarray(value, np.complex128),
                         halo_rows=halo)


def _oracle_grid(gu, gv, plane, value, n_u, n_v, n_w, kind, S, shape):
    b = {"gu": np.asarray(gu, float), "gv": np.asarray(gv, float),
         "plane": np.asarray(plane, np.uint32), "value": np.asarray(value, np.complex128),
         "v_start": 0, "v_count": n_v}
    return O.grid_slab(b, n_u, n_w, kind, S, shape)


def test_near_delta_kernel_hits_single_cell(W):
    spec = W.GridSpec(16, 16, 1, 1e-3)
    slab = W.slab_of(spec, 0, 1)
    out = W.ComplexGrid(spec, slab)
    W.grid_sector(_batch(W, spec, slab, [8.0], [8.0], [0], [1.0 + 0j], halo=1),
                  W.KernelSpec.gaussian(1, 1e-3), out)
    assert out.data[0, 8, 8] == pytest.approx(1.0)
    masked = out.data.copy()
    masked[0, 8, 8] = 0.0
    assert np.max(np.abs(masked)) < 1e-10


def test_on_center_record_closed_form_neighbourhood(W):
    spec = W.GridSpec(16, 16, 1, 1e-3)
    slab = W.slab_of(spec, 0, 1)
    out = W.ComplexGrid(spec, slab)
    W.grid_sector(_batch(W, spec, slab, [8.0], [8.0], [0], [(2 + 0j) * 0.5]),
                  W.KernelSpec.gaussian(3, 1.0), out)
    assert out.data[0, 8, 8] == pytest.approx(1.0, abs=1e-14)
    for j, i in ((7, 8), (9, 8), (8, 7), (8, 9)):
        assert out.data[0, j, i].real == pytest.approx(math.exp(-0.5), abs=1e-12)
    for j, i in ((7, 7), (9, 9), (7, 9), (9, 7)):
        assert out.data[0, j, i].real == pytest.approx(math.exp(-1.0), abs=1e-12)


def test_two_identical_records_double_the_grid(W):
    spec = W.GridSpec(16, 16, 2, 1e-3)
    slab = W.slab_of(spec, 0, 1)
    one, two = W.ComplexGrid(spec, slab), W.ComplexGrid(spec, slab)
    k = W.KernelSpec.gaussian(3, 1.0)
    W.grid_sector(_batch(W, spec, slab, [5.3], [7.8], [1], [1.5 - 0.5j]), k, one)
    W.grid_sector(_batch(W, spec, slab, [5.3, 5.3], [7.8, 7.8], [1, 1], [1.5 - 0.5j] * 2), k, two)
    assert np.allclose(two.data, 2.0 * one.data, rtol=0, atol=1e-15)


def test_record_outside_slab_halo_rejected(W):
    spec = W.GridSpec(16, 16, 1, 1e-3)
    slab = W.slab_of(spec, 0, 2)  # rows 0..7
    with pytest.raises(ValueError, match="outside slab"):
        _batch(W, spec, slab, [3.0], [14.0], [0], [1.0], halo=3)
    # and grid_sector itself applies the +-S predicate (gridder.py:198-199)
    b = _batch(W, spec, slab, [3.0], [11.5], [0], [1.0], halo=4)
    with pytest.raises(ValueError, match="outside slab"):
        W.grid_sector(b, W.KernelSpec.gaussian(3, 1.0), W.ComplexGrid(spec, slab))


def test_gridded_mass_matches_kernel_sums(W):
    spec = W.GridSpec(64, 64, 2, 1e-3)
    slab = W.slab_of(spec, 0, 1)
    out = W.ComplexGrid(spec, slab)
    rng = np.random.default_rng(3)
    n = 50
    gu, gv = rng.uniform(10, 54, n), rng.uniform(10, 54, n)
    value = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    W.grid_sector(_batch(W, spec, slab, gu, gv, rng.integers(0, 2, n), value),
                  W.KernelSpec.gaussian(3, 1.0), out)

    def footprint_sum(u, v):   # gridder.kernel_footprint_sum restated
        du = u - (np.floor(u) + np.arange(-3, 4))
        dv = v - (np.floor(v) + np.arange(-3, 4))
        du, dv = du[np.abs(du) <= 3], dv[np.abs(dv) <= 3]
        return float(O.kernel_value(O.KIND_GAUSSIAN, 3, 1.0, du[:, None], dv[None, :]).sum())

    expected = sum(val * footprint_sum(a, b) for a, b, val in zip(gu, gv, value))
    assert abs(out.data.sum() - expected) < 1e-10


def test_thread_count_independence_deterministic(W):
    spec = W.GridSpec(32, 32, 2, 1e-3)
    slab = W.slab_of(spec, 0, 1)
    rng = np.random.default_rng(9)
    n = 200
    b = _batch(W, spec, slab, rng.uniform(0, 32, n), rng.uniform(0, 32, n), rng.integers(0, 2, n),
               rng.standard_normal(n) + 1j * rng.standard_normal(n))
    k = W.KernelSpec.kaiser_bessel(3)
    outs = []
    for threads in (1, 2, 8):
        out = W.ComplexGrid(spec, slab)
        W.grid_sector(b, k, out, threads=threads, deterministic=True)
        outs.append(out.data.tobytes())
    assert outs[0] == outs[1] == outs[2]
    ref, _ = _oracle_grid(b.gu, b.gv, b.plane, b.value, 32, 32, 2, O.KIND_KAISER_BESSEL, 3,
                          k.shape_param)
    assert np.max(np.abs(np.frombuffer(outs[0], np.complex128).reshape(ref.shape) - ref)) <= 1e-12


def _dataset(n=1000, seed=11):
    src = ((0.01, -0.008, 2.0), (0.0, 0.0, 1.0))
    return Chunk(*O.generate_synthetic(src, n, 2, seed, n_time_slices=8, cell_size_lm=1e-3,
                                       w_max_native=12.0))


def _parts(chunk, R):
    from paper_2504_00959_b200.imager import _partition_bounds
    b, _ = _partition_bounds(chunk.time_index, R)
    return [chunk.rows(slice(lo, hi)) for lo, hi in b]


def _gather(slabs):
    return np.concatenate([s.data for s in slabs], axis=1)


def test_single_rank_equals_sequential_gridding(W):
    spec = W.GridSpec(64, 64, 4, 1e-3, w_max_native=12.0)
    c = _dataset()
    slabs, _ = W.grid_all([c], spec, W.KernelSpec.gaussian(3, 1.0), Topo(1, 1))
    prep = O.prepare(c.u, c.v, c.w, c.time_index, c.vis, c.weight, 64, 64, 4)
    ref, _ = _oracle_grid(prep["gu"], prep["gv"], prep["plane"], prep["value"], 64, 64, 4,
                          O.KIND_GAUSSIAN, 3, 1.0)
    assert np.max(np.abs(_gather(slabs) - ref)) <= 1e-12


def test_rank_counts_agree_bitwise_in_deterministic_mode(W):
    spec = W.GridSpec(64, 64, 4, 1e-3, w_max_native=12.0)
    c = _dataset()
    k = W.KernelSpec.gaussian(3, 1.0)
    imgs = {R: _gather(W.grid_all(_parts(c, R), spec, k, Topo(1, R))[0]) for R in (1, 2, 4)}
    assert imgs[1].tobytes() == imgs[2].tobytes() == imgs[4].tobytes()


def test_halo_records_counted_once_across_boundary(W):
    spec = W.GridSpec(32, 32, 1, 1e-3)
    k = W.KernelSpec.gaussian(3, 1.0)
    rng = np.random.default_rng(4)
    n = 40
    c = Chunk(rng.random(n), (15.7 + rng.random(n)) / 32.0, np.zeros(n),
              np.arange(n, dtype=np.uint32),
              (rng.standard_normal((n, 1)) + 1j * rng.standard_normal((n, 1))).astype(np.complex64),
              np.ones((n, 1), np.float32))
    one, _ = W.grid_all([c], spec, k, Topo(1, 1))
    two, _ = W.grid_all(_parts(c, 2), spec, k, Topo(1, 2))
    assert _gather(one).tobytes() == _gather(two).tobytes()


def test_concurrent_grid_all_within_tolerance(W):
    spec = W.GridSpec(64, 64, 4, 1e-3, w_max_native=12.0)
    c = _dataset()
    k = W.KernelSpec.gaussian(3, 1.0)
    det, _ = W.grid_all([c], spec, k, Topo(1, 1))
    conc, log = W.grid_all(_parts(c, 4), spec, k, Topo(2, 2, threads_per_rank=2),
                           Strategy("hybrid_ring", deterministic=False))
    assert np.max(np.abs(_gather(det) - _gather(conc))) <= 1e-12
    assert log.count(phase="exchange") == 12 and log.count(phase="reduce") > 0


# ---------------------------------------------------------------------------
# run_pipeline against the reference's own runs (tests/golden/pipeline.npz)
# ---------------------------------------------------------------------------

class SyntheticPowerMeter:
    """metrics.SyntheticPowerMeter (metrics.py:129-144) with its default watts."""
    watts = {"high": 500.0, "default": 500.0, "medium": 375.0, "low": 350.0}

    def joules(self, durations, freq_level):
        return {p: self.watts[freq_level] * s for p, s in durations.items()}


OPS = ("records", "grid_updates", "exchange_bytes", "reduce_bytes", "fft_bytes",
       "reduce_messages", "stack_pixels")


@pytest.mark.parametrize("name", ["t1x1", "t1x3", "t2x2h", "t2x3r", "t3x2d", "t1x4h", "t2x2r"])
def test_run_pipeline_matches_reference_runs(W, name, tmp_path):
    with np.load(GOLDEN / "pipeline.npz") as z:
        g = {k: z[k] for k in z.files if k.startswith(name + "_")}
    nn, rpn, det = (int(x) for x in g[f"{name}_topo"])
    res = W.run_pipeline(GOLDEN / "chunks.rvis", 64, 64, 4, 1e-3, W.KernelSpec.gaussian(3, 1.0),
                         topo=Topo(nn, rpn), strategy=Strategy(str(g[f"{name}_kind"]), bool(det)),
                         meter=SyntheticPowerMeter(), freq_level="medium", label=name,
                         out_dir=tmp_path)
    assert rel_l2(res.image.pixels, g[f"{name}_pixels"]) <= 1e-10
    assert dict(res.ops) == dict(zip(OPS, (int(x) for x in g[f"{name}_ops"])))
    assert (tmp_path / "messages.csv").read_text() == str(g[f"{name}_messages_csv"])
    assert sorted(res.run.energy_joules) == [str(x) for x in g[f"{name}_energy_keys"]]
    assert res.run.energy_joules["total"] == pytest.approx(
        sum(v for k, v in res.run.energy_joules.items() if k != "total"))
    assert sorted(res.run.phase_times) == ["fft", "gridding", "read", "reduce", "total",
                                           "wcorrect", "write"]
    assert res.paths["raw"].exists() and res.paths["sidecar"].exists()
    # bitwise reproducible run to run (bench.py:202-203 image-hash identity)
    again = W.run_pipeline(GOLDEN / "chunks.rvis", 64, 64, 4, 1e-3, W.KernelSpec.gaussian(3, 1.0),
                           topo=Topo(nn, rpn))
    assert again.image_sha256 == res.image_sha256


def test_run_pipeline_unsorted_dataset_raises(W, tmp_path):
    from paper_2504_00959_b200 import read_dataset, write_dataset
    h, c = read_dataset(GOLDEN / "chunks.rvis")
    c = dict(c)
    c["time_index"] = c["time_index"][::-1].copy()
    write_dataset(c, h, tmp_path / "bad.rvis")
    with pytest.raises(ValueError, match="sorted by time_index"):
        W.run_pipeline(tmp_path / "bad.rvis", 64, 64, 4, 1e-3, W.KernelSpec.gaussian(3, 1.0),
                       topo=Topo(1, 2))


def test_energy_counters_opt_in(W):
    """wsb_diag.gpu_joules / host_joules (NVML / RAPL around the call) are
    read only on request (WSB_EXEC_ENERGY); -1 / None otherwise."""
    from paper_2504_00959_b200 import read_dataset
    _, c = read_dataset(GOLDEN / "chunks.rvis")
    spec = W.GridSpec(64, 64, 4, 1e-3, w_max_native=40.0)
    k = W.KernelSpec.gaussian(3, 1.0)
    _, d0 = W.image(c["u"], c["v"], c["w"], c["time_index"], c["vis"], c["weight"], spec, k)
    assert d0["gpu_joules"] is None and d0["host_joules"] is None
    _, d1 = W.image(c["u"], c["v"], c["w"], c["time_index"], c["vis"], c["weight"], spec, k,
                    energy=True)
    assert d1["gpu_joules"] is not None and d1["gpu_joules"] >= 0.0
    assert d1["host_joules"] is None or d1["host_joules"] >= 0.0
    assert d1["exchanged_records"] == 0
