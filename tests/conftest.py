"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything
else runs on CPU (the driver runs ``-m "not gpu"`` here and ``-m gpu`` on a
B200).  The oracle (``oracle/``) is imported only as the checker."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and librbc.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def engine_cases():
    meta = json.loads((GOLDEN / "engine_cases.json").read_text())
    arrays = np.load(GOLDEN / "engine_cases.npz")
    return meta, {k: arrays[k] for k in arrays.files}


@pytest.fixture(scope="session")
def host_cases():
    arrays = np.load(GOLDEN / "host_cases.npz")
    return {k: arrays[k] for k in arrays.files}


def mode_for(label):
    from paper_1905_07439_b200.precision import parse_precision

    return parse_precision(label)


def case_levels(arrs, name, Q):
    return [(arrs[f"{name}/u{q}"], arrs[f"{name}/v{q}"], arrs[f"{name}/w{q}"]) for q in range(Q)]


def same_values(x, y) -> bool:
    """Value equality the reference's own tests use (np.array_equal: +0 == -0),
    plus equal dtype and shape."""
    x = np.asarray(x)
    y = np.asarray(y)
    return x.dtype == y.dtype and x.shape == y.shape and bool(np.array_equal(x, y))


def bit_equal(x, y) -> bool:
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    return x.dtype == y.dtype and x.shape == y.shape and x.tobytes() == y.tobytes()
