import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built libdrb200.so")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def golden(name):
    return np.load(GOLDEN / name)


def cfg_from(arr, **kw):
    from paper_2509_10466_b200 import DsttConfig
    w, h, p, c, k, heads, g = (int(v) for v in arr)
    return DsttConfig(width=w, height=h, patch=p, channels=c, kernel=k, heads=heads,
                      temporal_groups=g, **kw)


def perturb_1d(arrays, seed):
    """Same perturbation as make_golden.perturb_1d, in parameter order."""
    rng = np.random.default_rng(seed)
    out = []
    for a in arrays:
        if a.ndim == 1:
            a = (a + rng.normal(0.0, 0.1, a.shape).astype(np.float32)).astype(np.float32)
        out.append(a)
    return out


def digest(arrays):
    rows = []
    for a in arrays:
        a = np.asarray(a, np.float64).ravel()
        rows.append([a.sum(), (a * a).sum(), a[0]])
    return np.array(rows)


os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
