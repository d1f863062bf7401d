"""bc_matmul: the north-star argument list (U, V, W, depth, randomize flag,
seed, dtype) mapped onto the mirrored reference objects."""
import numpy as np
import pytest

import paper_1905_07439_b200 as rbc
from oracle import engine as oracle


def test_facade_argument_errors_without_a_gpu():
    f = rbc.strassen_formula()
    A = np.zeros((4, 4))
    with pytest.raises(ValueError):
        rbc.bc_matmul(A, A, f.u, f.v, f.w, depth=-1)
    with pytest.raises(ValueError):
        rbc.bc_matmul(A, A, f.u[:, :1], f.v, f.w, depth=1)  # not a bilinear formula
    with pytest.raises(ValueError):
        rbc.bc_matmul(A, A, f.u, f.v, f.w, depth=1, dtype="f128")


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f64", "f32", "f16"])
@pytest.mark.parametrize("randomize", [True, False])
def test_facade_equals_reference_objects_through_the_oracle(dtype, randomize):
    """Same seed, same plans: the facade's product equals the oracle's
    evaluation of the reference's objects (plans from derive_rng(seed, 2, trial,
    q), hatted tables with the 1/(1-kappa) rescale, or the plain formula)."""
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.precision import parse_precision

    mode = parse_precision(dtype)
    f = rbc.strassen_formula()
    g = np.random.default_rng(11)
    A, B = g.standard_normal((16, 16)), g.standard_normal((16, 16))
    depth, seed, trial = 3, 5, 2
    got = rbc.bc_matmul(A, B, f.u, f.v, f.w, depth, randomize=randomize, seed=seed, dtype=dtype,
                        trial=trial)
    a, b = mode.array(A)[None], mode.array(B)[None]
    if randomize:
        plans = [rbc.draw_plan(2, rbc.derive_rng(seed, rbc.ROLE_PLAN, trial, q)) for q in range(depth)]
        levels = [rbc.plan_levels(f, [p], mode) for p in plans]
    else:
        levels = [mode_tensors(f, mode)] * depth
    want = oracle.apply_levels(levels, a, b, mode)[0]
    assert got.dtype == want.dtype and np.array_equal(got, want)
    # depth 0 is the standard algorithm
    std = rbc.bc_matmul(A, B, f.u, f.v, f.w, 0, dtype=dtype)
    assert np.array_equal(std, oracle.leaf(a, b)[0])
