"""Generate tests/golden/rescale_cases.{npz,json} from the reference itself.

    python tests/golden/make_rescale_golden.py

Runs the unmodified reference ``randbc.rescale.rescaled_multiply``
(/root/reference/pkg/src/randbc/rescale.py:60-99, its engine numpy-only) on
seeded operands for several modes, formulas, depths and schedules, and
records inputs, outputs and the exceptions it raises.  binary16 goes through
the reference with this package's duck-typed HALF mode.  The
fixtures pin oracle/rescale.py (CPU tests) and the device rescaling
(tests/test_rescale_gpu.py); nothing at run time reads /root/reference.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

from randbc.formula import BilinearFormula, perturb, strassen_formula  # noqa: E402
from randbc.precision import DOUBLE, SINGLE  # noqa: E402
from randbc.rescale import DEFAULT_SCHEDULE, INSIDE, OUTSIDE, rescaled_multiply  # noqa: E402
from randbc.rng import derive_rng  # noqa: E402

from paper_1905_07439_b200.formula import load_formula  # noqa: E402
from paper_1905_07439_b200.precision import HALF  # noqa: E402

MODES = {"f64": DOUBLE, "f32": SINGLE, "f16": HALF}


def laderman():
    g = load_formula(ROOT / "paper_1905_07439_b200" / "formulas" / "laderman.txt")
    return BilinearFormula(g.u, g.v, g.w)


FORMULAS = {
    "strassen": strassen_formula,
    "laderman": laderman,
    "perturbed": lambda: perturb(strassen_formula(), 1e-3, 5, derive_rng(42)),
}
SCHEDULES = {
    "2xoi": DEFAULT_SCHEDULE,
    "o": (OUTSIDE,),
    "i": (INSIDE,),
    "none": (),
    "ioi": (INSIDE, OUTSIDE, INSIDE),
}
# name, mode, formula, Q, N, schedule, input kind
CASES = []
for mode in ("f64", "f32", "f16"):
    for sched in SCHEDULES:
        CASES.append((f"strassen_{mode}_{sched}", mode, "strassen", 3, 32, sched, "pos"))
    CASES.append((f"strassen_{mode}_2xoi_gauss", mode, "strassen", 2, 40, "2xoi", "gauss"))
    CASES.append((f"strassen_{mode}_2xoi_rows", mode, "strassen", 4, 48, "2xoi", "rows"))
    CASES.append((f"laderman_{mode}_2xoi", mode, "laderman", 2, 27, "2xoi", "gauss"))
    CASES.append((f"perturbed_{mode}_2xoi", mode, "perturbed", 2, 32, "2xoi", "gauss"))
    CASES.append((f"q0_{mode}_2xoi", mode, "strassen", 0, 20, "2xoi", "gauss"))
    CASES.append((f"zero_row_{mode}", mode, "strassen", 2, 16, "2xoi", "zero_row_a"))
    CASES.append((f"zero_col_{mode}", mode, "strassen", 2, 16, "2xoi", "zero_col_b"))
    CASES.append((f"zero_inside_row_{mode}", mode, "strassen", 2, 16, "i", "zero_row_b"))
CASES.append(("overflow_f16", "f16", "strassen", 2, 16, "none", "huge"))


def operands(kind, N, seed):
    g = derive_rng(seed)
    if kind == "pos":
        return g.random((N, N)) + 0.1, g.random((N, N)) + 0.1
    A, B = g.standard_normal((N, N)), g.standard_normal((N, N))
    if kind == "rows":
        A *= np.logspace(-3, 3, N)[:, None]
        B *= np.logspace(2, -2, N)[None, :]
    elif kind == "zero_row_a":
        A[3, :] = 0.0
    elif kind == "zero_col_b":
        B[:, 5] = 0.0
    elif kind == "zero_row_b":
        B[7, :] = 0.0
    elif kind == "huge":
        A *= 300.0
        B *= 300.0
    return A, B


def main():
    arrays, meta = {}, []
    for i, (name, mlabel, fname, Q, N, sched, kind) in enumerate(CASES):
        mode = MODES[mlabel]
        f = FORMULAS[fname]()
        A64, B64 = operands(kind, N, 1000 + i)
        A, B = mode.array(A64), mode.array(B64)
        raises, msg = None, None
        with np.errstate(all="ignore"):
            try:
                C = rescaled_multiply(A, B, Q, SCHEDULES[sched], mode, formula=f)
                arrays[f"{name}/out"] = C
            except (ValueError, OverflowError) as exc:
                raises, msg = type(exc).__name__, str(exc)
        arrays[f"{name}/a"] = A
        arrays[f"{name}/b"] = B
        meta.append(dict(name=name, mode=mlabel, formula=fname, Q=Q, N=N, schedule=sched,
                         kind=kind, raises=raises, message=msg))
    np.savez_compressed(HERE / "rescale_cases.npz", **arrays)
    (HERE / "rescale_cases.json").write_text(json.dumps(meta, indent=1))
    print(f"{len(meta)} rescale cases, {sum(m['raises'] is not None for m in meta)} raising")


if __name__ == "__main__":
    main()
