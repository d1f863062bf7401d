"""GPU: SURVEY §8f "next" rows -- plan-enumeration expectation
(randomize.py:293-334) and the rescaled 2x O-I baseline (rescale.py:60-99) --
against the CPU oracle restatement, plus the reference's own invariants."""

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
                                              ("f64", "perturbed", 4)])
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


@pytest.mark.parametrize("label", ["f32", "f64", "f16"])
def test_rescaled_multiply_matches_oracle(label):
    import paper_1905_07439_b200 as rbc
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.precision import parse_precision
    from paper_1905_07439_b200.rescale import DEFAULT_SCHEDULE, INSIDE, OUTSIDE, rescaled_multiply

    mode = parse_precision(label)
    g = rbc.derive_rng(40)
    A = mode.array(g.random((32, 32)) + 0.1)
    B = mode.array(g.random((32, 32)) + 0.1)
    f = rbc.strassen_formula()
    for schedule in (DEFAULT_SCHEDULE, (OUTSIDE,), (INSIDE,), ()):
        got = rescaled_multiply(A, B, 3, schedule, mode)
        # oracle: identical host scaling, oracle recursion
        import paper_1905_07439_b200.rescale as rs

        orig = rs.recursive_apply
        try:
            rs.recursive_apply = lambda f_, A_, B_, Q_, m_: oracle.apply_levels(
                [mode_tensors(f_, m_)] * Q_, A_[None], B_[None], m_)[0]
            want = rescaled_multiply(A, B, 3, schedule, mode)
        finally:
            rs.recursive_apply = orig
        assert np.array_equal(got, want), schedule
    assert np.array_equal(rescaled_multiply(A, B, 2, (), mode), rbc.recursive_apply(f, A, B, 2, mode))
    with pytest.raises(ValueError):
        rescaled_multiply(np.zeros((4, 4)), B[:4, :4], 1, DEFAULT_SCHEDULE, mode)
