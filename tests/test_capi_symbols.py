"""The C-ABI library loads (no GPU needed) and exports every symbol that
include/rbc.h declares; host-only entry points work without a device."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "rbc.h").read_text()
    return sorted(set(re.findall(r"\b(rbc_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1905_07439_b200 import _lib

    if not _lib.LIB_PATH.exists():
        from paper_1905_07439_b200.build import build

        build()
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    from paper_1905_07439_b200 import _lib

    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == syms


def test_abi_version(lib):
    assert lib.rbc_abi_version() == 1


def test_pack_plans_host_only(lib):
    from paper_1905_07439_b200 import engine

    perms = np.array([[[1, 0, 2], [2, 1, 0], [0, 2, 1]]])
    signs = np.array([[[1.0, -1.0, 1.0], [-1.0, -1.0, 1.0], [1.0, 1.0, -1.0]]])
    packed = engine.pack_plans(3, perms, signs)
    assert packed.shape == (1, 40)
    rec = packed[0].view(np.int8)
    perm = rec[0:12].reshape(3, 4)[:, :3]
    inv = rec[12:24].reshape(3, 4)[:, :3]
    neg = rec[24:36].reshape(3, 4)[:, :3]
    assert np.array_equal(perm, perms[0])
    for i in range(3):
        assert np.array_equal(inv[i][perms[0][i]], np.arange(3))
    assert np.array_equal(neg, (signs[0] < 0).astype(np.int8))
    with pytest.raises(ValueError):
        engine.pack_plans(3, np.array([[[0, 0, 1]] * 3]), np.ones((1, 3, 3)))
    with pytest.raises(ValueError):
        engine.pack_plans(3, perms, signs * 0.5)


def test_validation_before_device(lib):
    """Shape errors surface as ValueError even on a host without a GPU."""
    from paper_1905_07439_b200 import engine
    from paper_1905_07439_b200.precision import SINGLE

    one = np.ones((1, 4, 4), np.float32)
    with pytest.raises(ValueError, match="need at least one level"):
        engine.apply_levels([], one, one, SINGLE)
    u = np.ones((1, 7, 3, 3), np.float32)
    with pytest.raises(ValueError, match="not divisible"):
        engine.apply_levels([(u, u, u)], one, one, SINGLE)
    with pytest.raises(ValueError, match="inner dimensions"):
        engine.leaf_matmul(np.ones((1, 2, 3)), np.ones((1, 2, 3)), SINGLE)
    assert engine.leaf_matmul(np.ones((2, 3, 0)), np.ones((2, 0, 4)), SINGLE).shape == (2, 3, 4)


def test_no_silent_cpu_path_without_device(lib):
    from paper_1905_07439_b200 import _lib, engine
    from paper_1905_07439_b200.precision import SINGLE

    if lib.rbc_device_count() > 0:
        pytest.skip("a CUDA device is present")
    u = np.ones((1, 7, 2, 2), np.float32)
    one = np.ones((1, 4, 4), np.float32)
    with pytest.raises(RuntimeError):
        engine.apply_levels([(u, u, u)], one, one, SINGLE)
    with pytest.raises(RuntimeError):
        _lib.require_device()
