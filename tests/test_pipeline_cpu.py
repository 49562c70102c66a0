"""Host logic of the run_pipeline drop-in, CPU only: the virtual-topology
message log against the reference's own messages.csv (tests/golden/
pipeline.npz, written by the reference's run_pipeline), the time partition,
metrics.measure semantics, RunRecord rules and the energy meter."""

import sys
import types

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import wstack_oracle as O
from paper_2504_00959_b200 import energy, msglog
from paper_2504_00959_b200.imager import (RunRecord, MeterError, _partition_bounds, measure,
                                          read_dataset)

OPS = ("records", "grid_updates", "exchange_bytes", "reduce_bytes", "fft_bytes",
       "reduce_messages", "stack_pixels")


class Topo:
    def __init__(self, n_nodes, ranks_per_node, threads_per_rank=1):
        self.n_nodes, self.ranks_per_node, self.threads_per_rank = n_nodes, ranks_per_node, threads_per_rank

    @property
    def n_ranks(self):
        return self.n_nodes * self.ranks_per_node


@pytest.fixture(scope="module")
def golden_pipeline():
    with np.load(GOLDEN / "pipeline.npz") as z:
        return {k: z[k] for k in z.files}


def _counts(cols, n_v, S, bounds):
    """Exchange counts with the oracle's halo predicate (comms.py:521-523)."""
    R = len(bounds)
    gv = np.asarray(cols["v"], np.float64) * n_v
    out = []
    for lo, hi in bounds:
        out.append([int(O.halo_mask(gv[lo:hi], S, *O.partition_1d(n_v, R, d)).sum())
                    for d in range(R)])
    return out


@pytest.mark.parametrize("name", ["t1x1", "t1x3", "t2x2h", "t2x3r", "t3x2d", "t1x4h", "t2x2r"])
def test_virtual_log_matches_reference_messages(golden_pipeline, name, tmp_path):
    g = golden_pipeline
    nn, rpn, det = (int(x) for x in g[f"{name}_topo"])
    kind = str(g[f"{name}_kind"])
    topo = Topo(nn, rpn)
    _, cols = read_dataset(GOLDEN / "chunks.rvis")
    bounds, _ = _partition_bounds(cols["time_index"], topo.n_ranks)
    counts = _counts(cols, 64, 3, bounds)
    log = (msglog.virtual_log(topo, kind, 64, 64, 4, counts) if topo.n_ranks > 1
           else msglog.MessageLog())
    log.to_csv(tmp_path / "m.csv")
    assert (tmp_path / "m.csv").read_text() == str(g[f"{name}_messages_csv"])
    ops = dict(zip(OPS, (int(x) for x in g[f"{name}_ops"])))
    assert log.total_bytes(phase="exchange") == ops["exchange_bytes"]
    assert log.total_bytes(phase="reduce") == ops["reduce_bytes"]
    assert log.total_bytes(phase="fft") == ops["fft_bytes"]
    assert log.count(phase="reduce") == ops["reduce_messages"]


def test_partition_bounds_follow_reference_rules():
    t = np.repeat(np.arange(5, dtype=np.uint32), [3, 1, 4, 2, 5])
    b, ordered = _partition_bounds(t, 2)          # 5 slices -> (3, 2) slices
    assert ordered and b == [(0, 8), (8, 15)]
    b, ordered = _partition_bounds(t, 7)          # more ranks than slices: record runs
    assert not ordered and b[0] == (0, 3) and b[-1][1] == 15
    assert sum(hi - lo for lo, hi in b) == 15


def test_measure_adds_total_and_rejects_negative():
    class PhaseMeter:
        def joules(self, durations, freq_level):
            return {k: 2.0 * v for k, v in durations.items()}
    j = measure(PhaseMeter(), {"read": 1.0, "fft": 0.5})
    assert j == {"read": 2.0, "fft": 1.0, "total": 3.0}
    with pytest.raises(ValueError):
        measure(PhaseMeter(), {"read": -1.0})


def test_run_record_rules():
    ok = RunRecord("a", None, "default", {"read": 1.0, "total": 2.0}, {"total": 5.0})
    assert ok.total_seconds == 2.0 and ok.total_joules == 5.0 and ok.n_nodes == 1
    with pytest.raises(ValueError):
        RunRecord("a", None, "turbo", {"total": 1.0})
    with pytest.raises(ValueError):
        RunRecord("a", None, "default", {"read": 3.0, "total": 1.0})
    with pytest.raises(ValueError):
        RunRecord("a", None, "default", {"read": 1.0})
    with pytest.raises(ValueError):
        RunRecord("a", None, "default", {"total": 1.0}, {"total": -1.0})
    with pytest.raises(MeterError):
        RunRecord("a", None, "default", {"total": 1.0}).total_joules


def test_green_productivity_formula():
    # Eq. 4 (metrics.py:200-207): speedup / (alpha * relative energy); the
    # paper's GPU case: 95.9533 s / 60.8375 kJ vs 11.7309 s / 20.2325 kJ
    gp = energy.green_productivity(95.9533, 60837.5, 11.7309, 20232.5)
    assert abs(gp - 24.60) < 0.01
    assert energy.green_productivity(10, 10, 5, 5) == pytest.approx(4.0)
    assert energy.green_productivity(10, 10, 5, 5, alpha=2.0) == pytest.approx(2.0)
    with pytest.raises(ValueError):
        energy.green_productivity(1, 1, 1, 1, alpha=0)
    with pytest.raises(ValueError):
        energy.green_productivity(1, 0, 1, 1)


def test_nvml_rapl_meter_counter_wrap(tmp_path, monkeypatch):
    """GPU mJ from NVML (faked), host uJ from RAPL package counters with the
    wrap-around of max_energy_range_uj; sub-domains are not double counted."""
    pkg = tmp_path / "intel-rapl:0"
    sub = tmp_path / "intel-rapl:0:0"
    for d in (pkg, sub):
        d.mkdir()
    (pkg / "max_energy_range_uj").write_text("1000000\n")
    (pkg / "energy_uj").write_text("999000\n")
    (sub / "energy_uj").write_text("5\n")
    gpu = {"mj": 10_000}
    fake = types.SimpleNamespace(
        nvmlInit=lambda: None, nvmlDeviceGetCount=lambda: 1,
        nvmlDeviceGetHandleByIndex=lambda i: i,
        nvmlDeviceGetTotalEnergyConsumption=lambda h: gpu["mj"])
    monkeypatch.setitem(sys.modules, "pynvml", fake)
    monkeypatch.setattr(energy, "RAPL_ROOT", str(tmp_path))
    m = energy.NvmlRaplMeter(devices=[0])
    assert m.host_available
    m.start()
    gpu["mj"] = 12_500                                # +2.5 J
    (pkg / "energy_uj").write_text("4000\n")          # wrapped: +5000 uJ
    j = m.joules({"read": 1.0}, "default")
    assert j["gpu"] == pytest.approx(2.5)
    assert j["host"] == pytest.approx(0.005)
    assert j["total"] == pytest.approx(2.505)
    RunRecord("m", None, "default", {"total": 1.0}, j)      # numeric entries only


def test_modelled_host_meter_is_labelled_watts_times_seconds():
    m = energy.ModelledHostMeter(watts=400.0)
    j = m.joules({"read": 0.5, "fft": 1.5}, "default")
    assert j == {"read": 200.0, "fft": 600.0}
    assert "modelled" in m.source
    with pytest.raises(ValueError):
        energy.ModelledHostMeter(watts=0.0)
