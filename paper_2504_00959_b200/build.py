"""Build libwsb.so in-tree for sm_100a with nvcc (no JIT, no torch extension).

    python -m paper_2504_00959_b200.build [--force] [--verbose]

Objects go to build/ (git-ignored); the shared library lands next to this
file so it travels to the GPU box with the repository snapshot.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
LIB = PKG / "libwsb.so"
SOURCES = ["api.cu", "prepare.cu", "bucket.cu", "sort.cu", "grid.cu", "fft.cu", "peer.cu"]
HEADERS = ["wsb_internal.cuh", "i0_coeffs.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def stale_sources(lib: Path = LIB) -> list:
    """Sources / headers newer than ``lib`` (names), [] if it is current."""
    if not lib.exists():
        return ["(missing)"]
    t = lib.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS] + [ROOT / "include" / "wsb.h"]
    return [d.name for d in deps if d.exists() and d.stat().st_mtime > t]


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> Path:
    """debug: device bounds checks (WSB_DCHECK) into libwsb_dbg.so / build/dbg."""
    nvcc = _nvcc()
    build_dir = BUILD / "dbg" if debug else BUILD
    lib = PKG / "libwsb_dbg.so" if debug else LIB
    flags = FLAGS + (["-DWSB_DEBUG_CHECKS"] if debug else [])
    build_dir.mkdir(parents=True, exist_ok=True)
    hdrs = [CSRC / h for h in HEADERS] + [ROOT / "include" / "wsb.h"]
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = build_dir / (Path(src).stem + ".o")
        objs.append(o)
        if force or _stale(o, [s, *hdrs]):
            cmd = [nvcc, *ARCH, *flags, "-I", str(ROOT / "include"), "-c", str(s), "-o", str(o)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            log = (build_dir / (Path(src).stem + ".ptxas.log"))
            log.write_text(r.stdout + r.stderr)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stdout.write(r.stderr)
    if force or _stale(lib, objs):
        tmp = lib.with_suffix(".so.tmp")
        cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
        tmp.replace(lib)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--debug", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose, a.debug))
