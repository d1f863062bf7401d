"""GPU: SURVEY §8f "next" row 3 -- plan-enumeration expectation
(randomize.py:293-334) -- against the CPU oracle restatement, plus the
reference's own invariants.  Row 2 (rescaling) is tests/test_rescale_gpu.py."""

import itertools

import numpy as np
import pytest

from oracle import engine as oracle

pytestmark = pytest.mark.gpu


def _oracle_expectation(f, A, B, mode):
    from paper_1905_07439_b200.randomize import _all_plans, plan_levels

    total = np.zeros(A.shape)
    count = 0
    plans = list(_all_plans(f.n))
    for chunk in range(0, len(plans), 97):  # any chunking: values are per plan
        batch = plans[chunk:chunk + 97]
        C = oracle.apply_levels([plan_levels(f, batch, mode)], A[None], B[None], mode)
        for t in range(C.shape[0]):
            np.add(total, C[t].astype(np.float64), out=total)
            count += 1
    return total / float(count)


@pytest.mark.parametrize("label,which,size", [("f64", "strassen", 4), ("f32", "strassen", 6),
                                              ("f64", "perturbed", 4), ("f32", "perturbed", 6),
                                              ("f16", "perturbed", 4)])
def test_enumerate_expectation_matches_oracle(label, which, size):
    import paper_1905_07439_b200 as rbc
    from paper_1905_07439_b200.precision import parse_precision
    from paper_1905_07439_b200.randomize import enumerate_expectation

    mode = parse_precision(label)
    f = rbc.strassen_formula() if which == "strassen" else rbc.perturb(
        rbc.strassen_formula(), 1e-3, 5, rbc.derive_rng(42))
    g = rbc.derive_rng(35, size)
    A = mode.array(g.standard_normal((size, size)))
    B = mode.array(g.standard_normal((size, size)))
    got = enumerate_expectation(f, A, B, mode)
    small = enumerate_expectation(f, A, B, mode, chunk_elements=16)
    want = _oracle_expectation(f, A, B, mode)
    assert np.array_equal(got, want)
    assert np.array_equal(small, got)  # chunking neutral (reference test_randomize.py:316-322)
    if which == "strassen" and label == "f64":
        # unbiasedness of an exact formula (reference test_randomize.py:285-296)
        ref = A @ B
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-13




@pytest.mark.parametrize("label,N", [("f64", 3), ("f32", 6)])
def test_enumerate_expectation_laderman_110592_plans(label, N):
    """n = 3 (Laderman, (2^3)^3 (3!)^3 = 110,592 plans, under the reference's
    10^6 budget, randomize.py:293-334): the device enumeration equals the
    oracle's sequential binary64 average in enumeration order, bit for bit,
    and (binary64) the exact formula's expectation is A @ B to rounding."""
    import time

    import paper_1905_07439_b200 as rbc
    from paper_1905_07439_b200.precision import parse_precision
    from paper_1905_07439_b200.randomize import _hatted_batch, all_plan_arrays, enumerate_expectation

    mode = parse_precision(label)
    f = rbc.laderman_formula()
    g = rbc.derive_rng(36, N)
    A = mode.array(g.standard_normal((N, N)))
    B = mode.array(g.standard_normal((N, N)))
    t0 = time.perf_counter()
    got = enumerate_expectation(f, A, B, mode)
    dt = time.perf_counter() - t0
    perms, signs = all_plan_arrays(3)
    total = np.zeros((N, N))
    for c0 in range(0, len(perms), 8192):
        lv = _hatted_batch(f, perms[c0:c0 + 8192], signs[c0:c0 + 8192], mode)
        C = oracle.apply_levels([lv], A[None], B[None], mode)
        for t in range(C.shape[0]):
            np.add(total, C[t].astype(np.float64), out=total)
    want = total / float(len(perms))
    assert np.array_equal(got, want)
    print(f"110,592-plan enumeration on the GPU: {dt:.2f} s")
    if label == "f64":
        # unbiasedness of an exact formula, up to the rounding of a
        # sequential sum of 110,592 products (~count * u relative)
        ref = A @ B
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-10
