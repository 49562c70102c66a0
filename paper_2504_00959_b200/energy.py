"""Energy-to-solution meter: NVML on the GPUs + RAPL on the host.

Same duck type as the reference's PlatformCounterMeter (metrics.py:147-180):
``start()`` latches the counters, ``joules(durations, freq_level)`` returns
``{"total": J, ...}`` for the window since ``start()``. GPU energy comes from
``nvmlDeviceGetTotalEnergyConsumption`` (mJ, per device); host energy from
``/sys/class/powercap/intel-rapl:*/energy_uj`` package counters when they
are readable (they are absent in some containers: the host part is then
reported as None and ``total`` is the GPU energy alone, flagged by
``host_available``). ``green_productivity`` is the paper's Eq. 4 exactly as
metrics.py:200-207 computes it.
"""

from __future__ import annotations

import glob
from pathlib import Path


RAPL_ROOT = "/sys/class/powercap"

# Host power model used when RAPL is unreadable: the reference's synthetic
# meter default for a CPU node at the OS-governed frequency
# (metrics.py:56-57, DEFAULT_WATTS["default"]).
MODELLED_HOST_WATTS = 500.0


def _rapl_domains():
    doms = []
    for d in sorted(glob.glob(f"{RAPL_ROOT}/intel-rapl:*")):
        if ":" in Path(d).name[len("intel-rapl:"):]:
            continue                      # sub-domains (core, uncore, dram) are inside the package
        e = Path(d) / "energy_uj"
        m = Path(d) / "max_energy_range_uj"
        try:
            int(e.read_text())
            doms.append((e, int(m.read_text()) if m.exists() else 2 ** 32))
        except (OSError, ValueError):
            pass
    return doms


class NvmlRaplMeter:
    def __init__(self, devices=None, host: bool = True):
        import pynvml
        self._nv = pynvml
        pynvml.nvmlInit()
        n = pynvml.nvmlDeviceGetCount()
        idx = range(n) if devices is None else devices
        self.handles = [pynvml.nvmlDeviceGetHandleByIndex(int(i)) for i in idx]
        self.rapl = _rapl_domains() if host else []
        self._g0 = self._h0 = None

    @property
    def host_available(self) -> bool:
        return bool(self.rapl)

    def _gpu_mj(self):
        return [self._nv.nvmlDeviceGetTotalEnergyConsumption(h) for h in self.handles]

    def _host_uj(self):
        return [int(e.read_text()) for e, _ in self.rapl]

    def start(self):
        self._g0 = self._gpu_mj()
        self._h0 = self._host_uj()

    def joules(self, durations=None, freq_level: str = "default") -> dict:
        if self._g0 is None:
            self.start()
        g1, h1 = self._gpu_mj(), self._host_uj()
        gpu = sum(b - a for a, b in zip(self._g0, g1)) / 1e3
        host = None
        if self.rapl:
            host = 0.0
            for (e, wrap), a, b in zip(self.rapl, self._h0, h1):
                host += ((b - a) % wrap) / 1e6
        self._g0 = self._h0 = None
        out = {"total": gpu + (host or 0.0), "gpu": gpu}
        if host is not None:          # RunRecord rejects non-numeric entries
            out["host"] = host
        return out


class ModelledHostMeter:
    """Host energy as watts x seconds per phase -- the reference's
    SyntheticPowerMeter model (metrics.py:129-144) at one power level, used
    (and labelled as modelled) only where RAPL cannot be read."""

    def __init__(self, watts: float = MODELLED_HOST_WATTS):
        if watts <= 0:
            raise ValueError(f"watts must be positive, got {watts}")
        self.watts = float(watts)
        self.source = f"modelled host power {self.watts:.0f} W (SyntheticPowerMeter default level)"

    def start(self):
        pass

    def joules(self, durations: dict, freq_level: str = "default") -> dict:
        return {phase: self.watts * seconds for phase, seconds in durations.items()}


def green_productivity(t_ref: float, e_ref: float, t_test: float, e_test: float,
                       alpha: float = 1.0) -> float:
    """GP = (t_ref / t_test) / (alpha * e_test / e_ref) (metrics.py:200-207)."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    if min(t_ref, e_ref, t_test, e_test) <= 0:
        raise ValueError("times and energies must be positive")
    return (t_ref / t_test) / (alpha * e_test / e_ref)
