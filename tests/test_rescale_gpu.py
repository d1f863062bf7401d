"""GPU: the device-resident rescaling baseline (rbc_rescaled_multiply, kernels
in csrc/rescale.cu; reference rescale.py:60-99) against the reference's own
outputs (tests/golden/rescale_cases.*) and the independent CPU oracle
(oracle/rescale.py), bit for bit, including its exceptions."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, mode_for
from oracle import rescale as oracle_rescale
from test_oracle_rescale import SCHED, formula_tables

pytestmark = pytest.mark.gpu

CASES = json.loads((GOLDEN / "rescale_cases.json").read_text())


@pytest.fixture(scope="module")
def arrays():
    z = np.load(GOLDEN / "rescale_cases.npz")
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_device_rescale_matches_reference(case, arrays):
    from paper_1905_07439_b200 import _lib
    from paper_1905_07439_b200.rescale import rescaled_multiply

    _lib.require_device()
    mode = mode_for(case["mode"])
    f, _ = formula_tables(case["formula"], mode)
    a, b = arrays[case["name"] + "/a"], arrays[case["name"] + "/b"]
    args = (a, b, case["Q"], SCHED[case["schedule"]], mode, f)
    if case["raises"] == "ValueError":
        with pytest.raises(ValueError, match=case["message"]):
            rescaled_multiply(*args)
        return
    if case["raises"] == "OverflowError":
        with pytest.raises(OverflowError, match="result left the half range"):
            rescaled_multiply(*args)
        return
    got = rescaled_multiply(*args)
    want = arrays[case["name"] + "/out"]
    assert got.dtype == want.dtype and np.array_equal(got, want), case["name"]


@pytest.mark.parametrize("label", ["f64", "f32", "f16"])
@pytest.mark.parametrize("N,Q", [(64, 3), (96, 5), (256, 2)])
def test_device_rescale_matches_oracle(label, N, Q):
    """Larger sizes than the fixtures (and N=96: 3 * 2^5) against the CPU
    oracle: the default 2x O-I schedule on graded inputs."""
    from paper_1905_07439_b200 import strassen_formula
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.rescale import DEFAULT_SCHEDULE, rescaled_multiply
    from paper_1905_07439_b200.rng import derive_rng

    mode = mode_for(label)
    g = derive_rng(7, N, Q)
    A = mode.array(g.standard_normal((N, N)) * np.logspace(-2, 2, N)[:, None])
    B = mode.array(g.standard_normal((N, N)) * np.logspace(1, -1, N)[None, :])
    f = strassen_formula()
    u, v, w = (t[0] for t in mode_tensors(f, mode))
    got = rescaled_multiply(A, B, Q, DEFAULT_SCHEDULE, mode, f)
    want = oracle_rescale.rescaled_multiply(A, B, Q, DEFAULT_SCHEDULE, mode, u, v, w)
    assert np.array_equal(got, want, equal_nan=True)
