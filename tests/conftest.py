import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")


def _load(name):
    with np.load(GOLDEN / name) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_bucket():
    return _load("bucket.npz")


@pytest.fixture(scope="session")
def golden_grid():
    return _load("grid.npz")


@pytest.fixture(scope="session")
def golden_image():
    return _load("image.npz")


def chunk_from(g, prefix):
    return (g[prefix + "u"], g[prefix + "v"], g[prefix + "w"], g[prefix + "time_index"],
            g[prefix + "vis"], g[prefix + "weight"])


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))
