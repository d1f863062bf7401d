"""Pin the CPU oracle against fixtures produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import bit_equal, case_levels, mode_for
from oracle import engine as oracle


def test_engine_cases_bitwise(engine_cases):
    meta, arrs = engine_cases
    assert len(meta["engine"]) >= 20
    for case in meta["engine"]:
        name = case["name"]
        mode = mode_for(case["mode"])
        levels = case_levels(arrs, name, case["Q"])
        a, b = arrs[f"{name}/a"], arrs[f"{name}/b"]
        stats = {}
        if case["raises"] == "OverflowError":
            with np.errstate(all="ignore"), pytest.raises(OverflowError):
                oracle.apply_levels(levels, a, b, mode, stats)
            continue
        out = oracle.apply_levels(levels, a, b, mode, stats)
        assert bit_equal(out, arrs[f"{name}/out"]), name
        assert stats["leaf_multiplies"] == case["leaf_multiplies"], name


def test_leaf_cases_bitwise(engine_cases):
    meta, arrs = engine_cases
    for case in meta["leaf"]:
        name = case["name"]
        out = oracle.leaf(arrs[f"{name}/x"], arrs[f"{name}/y"])
        assert bit_equal(out, arrs[f"{name}/out"]), name


def test_summation_order_pin(engine_cases):
    # reference test_multiply.py:76-81: (1 + 1e-16) - 1 in binary64
    _, arrs = engine_cases
    assert arrs["L10_f64_order/out"].ravel()[0] == (1.0 + 1e-16) - 1.0


def test_oracle_errors():
    from paper_1905_07439_b200.precision import SINGLE

    with pytest.raises(ValueError):
        oracle.apply_levels([], np.ones((1, 2, 2)), np.ones((1, 2, 2)), SINGLE)
    u = np.ones((1, 7, 2, 2), dtype=np.float32)
    with pytest.raises(ValueError):
        oracle.apply_levels([(u, u, u)], np.ones((1, 3, 3), np.float32),
                            np.ones((1, 3, 3), np.float32), SINGLE)
    with pytest.raises(ValueError):
        oracle.leaf(np.ones((1, 2, 3)), np.ones((1, 2, 3)))
