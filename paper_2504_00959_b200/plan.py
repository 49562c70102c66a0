"""Benchmark campaigns in the reference's format (bench.py:44-205): a plan
sweeps topologies x strategies x frequency levels over one dataset, runs
each cell ``repeats`` times through ``run_pipeline`` and writes
``runs_raw.csv`` (one row per run) and ``runs_aggregate.csv`` (mean and
sample standard deviation per cell, and whether the image hashes of the
repeats are identical) with the reference's column names, so existing
report tooling reads them unchanged. A failed run aborts its cell, is
recorded with its reason and never poisons the aggregates."""

from __future__ import annotations

import csv
import itertools
import statistics
from dataclasses import dataclass, field
from pathlib import Path

from .imager import OPS_COLUMNS, run_pipeline

PHASES = ("read", "gridding", "reduce", "fft", "wcorrect", "write")   # metrics.PHASES
PHASE_COLUMNS = [f"{p}_s" for p in PHASES] + ["total_s"]
RAW_COLUMNS = (["config", "label", "topology", "threads", "strategy", "deterministic",
                "freq_level", "repeat", "status", "failure_reason", "image_sha256"]
               + PHASE_COLUMNS + ["total_j"] + list(OPS_COLUMNS))
TIMING_COLUMNS = PHASE_COLUMNS + ["total_j"]


@dataclass
class BenchPlan:
    """One campaign over a dataset file (the reference's BenchPlan fields;
    ``topologies`` / ``strategies`` label the cells -- the GPU path has no
    virtual ranks and is always deterministic)."""
    n_u: int
    n_v: int
    n_w: int
    cell_size_lm: float
    kernel: object
    topologies: list
    strategies: list
    freq_levels: list = field(default_factory=lambda: ["default"])
    repeats: int = 4
    dataset: Path | None = None
    meter: object | None = None
    output_dir: Path = Path("bench_out")

    def __post_init__(self):
        if self.repeats < 1:
            raise ValueError("repeats must be >= 1")
        if not self.topologies or not self.strategies or not self.freq_levels:
            raise ValueError("sweep lists must be non-empty")
        if self.dataset is None:
            raise ValueError("a dataset path is required (write one with write_dataset)")


@dataclass
class PlanResult:
    raw_rows: list
    aggregate_rows: list
    aggregate_header: list
    raw_path: Path
    aggregate_path: Path
    all_ok: bool


def _label(topo, strategy, freq) -> str:
    t = topo.label() if hasattr(topo, "label") else str(topo)
    threads = getattr(topo, "threads_per_rank", 1)
    kind = getattr(strategy, "kind", str(strategy))
    return f"{t}t{threads}_{kind}_{freq}"


def _fmt(v):
    return f"{v:.10g}" if isinstance(v, float) else v


def mean_std(values) -> tuple[float, float]:
    values = list(values)
    m = statistics.fmean(values)
    return m, (statistics.stdev(values) if len(values) > 1 else 0.0)


def aggregate_rows(raw_rows):
    """Per-configuration mean and sample stddev over the successful repeats
    (bench.py:180-205)."""
    stat_cols = PHASE_COLUMNS + ["total_j"] + list(OPS_COLUMNS)
    header = ["config", "label", "status", "n_ok", "failure_reason"]
    for col in stat_cols:
        header += [f"{col}_mean", f"{col}_std"]
    header += ["image_hashes_identical"]
    by_config: dict = {}
    for row in raw_rows:
        by_config.setdefault(row["config"], []).append(row)
    out = []
    for config in sorted(by_config):
        rows = by_config[config]
        ok = [r for r in rows if r["status"] == "ok"]
        failed = [r for r in rows if r["status"] != "ok"]
        line = [config, rows[0]["label"], "ok" if not failed else "failed", len(ok),
                failed[0]["failure_reason"] if failed else ""]
        for col in stat_cols:
            m, s = mean_std([float(r[col]) for r in ok]) if ok else (0.0, 0.0)
            line += [m, s]
        line += [int(len({r["image_sha256"] for r in ok}) <= 1)]
        out.append(line)
    return header, out


def run_plan(plan: BenchPlan, device: int = 0) -> PlanResult:
    out_dir = Path(plan.output_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    raw_rows = []
    cells = list(itertools.product(plan.topologies, plan.strategies, plan.freq_levels))
    for ci, (topo, strategy, freq) in enumerate(cells):
        label = _label(topo, strategy, freq)
        for rep in range(plan.repeats):
            base = {"config": ci, "label": label,
                    "topology": topo.label() if hasattr(topo, "label") else str(topo),
                    "threads": getattr(topo, "threads_per_rank", 1),
                    "strategy": getattr(strategy, "kind", str(strategy)),
                    "deterministic": int(getattr(strategy, "deterministic", True)),
                    "freq_level": freq, "repeat": rep}
            try:
                res = run_pipeline(plan.dataset, plan.n_u, plan.n_v, plan.n_w, plan.cell_size_lm,
                                   kernel=plan.kernel, topo=topo, strategy=strategy,
                                   meter=plan.meter, freq_level=freq, label=label, device=device)
            except Exception as exc:  # the cell aborts, the plan continues
                raw_rows.append({**base, "status": "failed",
                                 "failure_reason": f"{type(exc).__name__}: {exc}",
                                 "image_sha256": ""})
                break
            row = {**base, "status": "ok", "failure_reason": "", "image_sha256": res.image_sha256}
            for p in PHASES:
                row[f"{p}_s"] = res.run.phase_times.get(p, 0.0)
            row["total_s"] = res.run.phase_times.get("total", 0.0)
            row["total_j"] = res.run.energy_joules.get("total", 0.0)
            row.update(res.ops)
            raw_rows.append(row)
    raw_path = out_dir / "runs_raw.csv"
    with open(raw_path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=RAW_COLUMNS, restval="")
        w.writeheader()
        for row in raw_rows:
            w.writerow({k: _fmt(row.get(k, "")) for k in RAW_COLUMNS})
    agg_header, agg_rows = aggregate_rows(raw_rows)
    agg_path = out_dir / "runs_aggregate.csv"
    with open(agg_path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(agg_header)
        for row in agg_rows:
            w.writerow([_fmt(v) for v in row])
    return PlanResult(raw_rows=raw_rows, aggregate_rows=agg_rows, aggregate_header=agg_header,
                      raw_path=raw_path, aggregate_path=agg_path,
                      all_ok=all(r["status"] == "ok" for r in raw_rows))
