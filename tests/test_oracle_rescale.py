"""CPU: pin oracle/rescale.py (the independent restatement of the reference's
rescaled_multiply, rescale.py:36-99) bitwise against outputs of the
reference itself (tests/golden/rescale_cases.*, make_rescale_golden.py)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, mode_for
from oracle import rescale as oracle_rescale

CASES = json.loads((GOLDEN / "rescale_cases.json").read_text())
SCHED = {"2xoi": ("outside", "inside", "outside", "inside"), "o": ("outside",),
         "i": ("inside",), "none": (), "ioi": ("inside", "outside", "inside")}


@pytest.fixture(scope="module")
def arrays():
    z = np.load(GOLDEN / "rescale_cases.npz")
    return {k: z[k] for k in z.files}


def formula_tables(name, mode):
    from paper_1905_07439_b200 import formula as fm
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.rng import derive_rng

    f = {"strassen": fm.strassen_formula, "laderman": fm.laderman_formula,
         "perturbed": lambda: fm.perturb(fm.strassen_formula(), 1e-3, 5, derive_rng(42))}[name]()
    return f, [t[0] for t in mode_tensors(f, mode)]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_rescale_matches_reference(case, arrays):
    mode = mode_for(case["mode"])
    _, (u, v, w) = formula_tables(case["formula"], mode)
    a, b = arrays[case["name"] + "/a"], arrays[case["name"] + "/b"]
    args = (a, b, case["Q"], SCHED[case["schedule"]], mode, u, v, w)
    if case["raises"] == "ValueError":
        with pytest.raises(ValueError, match=case["message"]):
            oracle_rescale.rescaled_multiply(*args)
        return
    if case["raises"] == "OverflowError":
        with pytest.raises(OverflowError):
            oracle_rescale.rescaled_multiply(*args)
        return
    got = oracle_rescale.rescaled_multiply(*args)
    want = arrays[case["name"] + "/out"]
    assert got.dtype == want.dtype and got.tobytes() == want.tobytes(), case["name"]
