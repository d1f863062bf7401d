"""Reproduce rows of the reference artifact pkg/artifacts/s2-variants-320.csv
(`randbc experiment s2-variants --seed 1`, f32, n=320, Q=1..5, 100 plans)
from the seed layout alone (reference experiments.py:237-261, 327-379).

GPU test: every gaussian and adv1 row of the standard, deterministic,
full_random, sign_only and perm_only algorithms, through this package's L2
API on the B200.  CPU test: a subset through the oracle, pinning the host
mirror (seeds, matrices, plans, variants) independently of the GPU.

Tolerance: 1e-12 relative (SURVEY §8c gate).  C and the binary64 truth are
bit-identical to the reference's; the remaining differences are the
platform-dependent ulps of the Frobenius norms.
"""

from collections import defaultdict
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden" / "s2_variants_320.csv"
RTOL = 1e-12
VARIANT = {"full_random": "full", "sign_only": "sign", "perm_only": "perm"}


def load_rows():
    rows = defaultdict(dict)
    lines = GOLDEN.read_text().splitlines()
    for ln in lines[1:]:
        exp, alg, kind, n, Q, trial, seed, rel, running = ln.split(",")
        rows[(kind, alg, int(Q))][int(trial)] = float(rel)
    return rows


def prepare(kind):
    from paper_1905_07439_b200 import DOUBLE, SINGLE, MatrixSpec, derive_seed, generate
    from paper_1905_07439_b200.matgen import MATRIX_KINDS

    mseed = derive_seed(1, 1, 0, MATRIX_KINDS.index(kind))
    A64, B64 = generate(MatrixSpec(kind, 320, mseed))
    Am, Bm = SINGLE.array(A64), SINGLE.array(B64)
    return Am, Bm, DOUBLE


def frob(x):
    return float(np.linalg.norm(np.asarray(x, dtype=np.float64).ravel()))


def rel_errors(results, ref, refnorm):
    res = np.asarray(results, dtype=np.float64)
    diff = res - ref[None]
    return np.sqrt(np.sum(diff * diff, axis=(1, 2))) / refnorm


def trial_plans(Q, trials, variant):
    from paper_1905_07439_b200 import RecursivePlan, derive_rng, draw_plan, variant_plan

    out = []
    for t in trials:
        levels = tuple(draw_plan(2, derive_rng(1, 2, t, q)) for q in range(Q))
        out.append(RecursivePlan(tuple(variant_plan(p, variant) for p in levels)))
    return out


def test_golden_subset_cpu_oracle():
    """Oracle + host mirror reproduce the artifact: Q=1,2, first 3 trials."""
    from oracle import engine as oracle
    from paper_1905_07439_b200 import SINGLE, strassen_formula
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.randomize import plan_levels

    rows = load_rows()
    f = strassen_formula()
    Am, Bm, _ = prepare("gaussian")
    ref = oracle.standard_multiply(Am.astype(np.float64), Bm.astype(np.float64))
    refnorm = frob(ref)
    std = oracle.standard_multiply(Am, Bm)
    assert frob(std.astype(np.float64) - ref) / refnorm == pytest.approx(
        rows[("gaussian", "standard", 0)][0], rel=RTOL)
    for Q in (1, 2):
        det = oracle.apply_levels([mode_tensors(f, SINGLE)] * Q, Am[None], Bm[None], SINGLE)[0]
        assert frob(det.astype(np.float64) - ref) / refnorm == pytest.approx(
            rows[("gaussian", "deterministic", Q)][0], rel=RTOL)
        for alg, var in VARIANT.items():
            rplans = trial_plans(Q, (1, 2, 3), var)
            levels = [plan_levels(f, [rp.levels[q] for rp in rplans], SINGLE) for q in range(Q)]
            C = oracle.apply_levels(levels, Am[None], Bm[None], SINGLE)
            got = rel_errors(C, ref, refnorm)
            want = [rows[("gaussian", alg, Q)][t] for t in (1, 2, 3)]
            np.testing.assert_allclose(got, want, rtol=RTOL, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["gaussian", "uniform", "adv1", "adv2", "adv3", "hilbert"])
def test_golden_rows_gpu(kind):
    from paper_1905_07439_b200 import (
        DOUBLE,
        SINGLE,
        recursive_apply,
        recursive_randomized_apply_many,
        standard_multiply,
        strassen_formula,
    )

    rows = load_rows()
    f = strassen_formula()
    Am, Bm, _ = prepare(kind)
    ref = standard_multiply(Am.astype(np.float64), Bm.astype(np.float64), DOUBLE)
    refnorm = frob(ref)
    std = standard_multiply(Am, Bm, SINGLE)
    assert frob(std.astype(np.float64) - ref) / refnorm == pytest.approx(
        rows[(kind, "standard", 0)][0], rel=RTOL)
    from paper_1905_07439_b200.rescale import DEFAULT_SCHEDULE, rescaled_multiply

    checked = 1
    for Q in range(1, 6):
        det = recursive_apply(f, Am, Bm, Q, SINGLE)
        assert frob(det.astype(np.float64) - ref) / refnorm == pytest.approx(
            rows[(kind, "deterministic", Q)][0], rel=RTOL)
        resc = rescaled_multiply(Am, Bm, Q, DEFAULT_SCHEDULE, SINGLE)
        assert frob(resc.astype(np.float64) - ref) / refnorm == pytest.approx(
            rows[(kind, "rescaled_2xoi", Q)][0], rel=RTOL)
        checked += 2
        for alg, var in VARIANT.items():
            rplans = trial_plans(Q, range(1, 101), var)
            C = recursive_randomized_apply_many(f, rplans, Am, Bm, SINGLE)
            got = rel_errors(C, ref, refnorm)
            want = [rows[(kind, alg, Q)][t] for t in range(1, 101)]
            np.testing.assert_allclose(got, want, rtol=RTOL, atol=0)
            checked += 100
    assert checked == 1 + 5 * 302
