"""Seeded differential tests: random engine problems (shapes, grids, ranks,
depths, trial layouts, coefficient kinds, special values) through the drop-in
entry points against the CPU oracle.  The dense-coefficient kernels must be
bit-identical (signed zeros included); with plan recognition on, recognised
+-1 tables run on the plan kernels, whose contract is value equality
(DESIGN section 2)."""

import numpy as np
import pytest

from conftest import mode_for, same_values
from oracle import engine as oracle

pytestmark = pytest.mark.gpu

LABELS = ("f64", "f32", "f16")


@pytest.fixture(scope="module")
def eng():
    from paper_1905_07439_b200 import _lib, engine

    _lib.require_device()
    return engine


def _coeffs(g, mode, Tc, R, n, kind):
    if kind == "pm1":  # sparse +-1 / 0 entries, signed zeros included
        c = g.choice([-1.0, 0.0, 0.0, 1.0], size=(Tc, R, n, n))
        c[g.random(c.shape) < 0.1] = -0.0
    elif kind == "small_int":
        c = g.integers(-3, 4, size=(Tc, R, n, n)).astype(np.float64)
    else:
        c = g.standard_normal((Tc, R, n, n))
    return mode.array(c)


def _operand(g, mode, T0, N):
    x = g.standard_normal((T0, N, N))
    x[g.random(x.shape) < 0.05] = 0.0
    x[g.random(x.shape) < 0.02] = -0.0
    return mode.array(x)


def _problem(seed):
    g = np.random.default_rng(1000 + seed)
    label = LABELS[seed % 3]
    mode = mode_for(label)
    n = int(g.choice([2, 2, 3, 3, 4]))
    Q = int(g.integers(1, 4 if n < 4 else 3))
    m = int(g.integers(1, 6))
    N = m * n ** Q
    T = int(g.integers(1, 5))
    T0 = int(g.choice([1, T]))
    kind = str(g.choice(["pm1", "small_int", "gauss"]))
    levels = []
    for _ in range(Q):
        R = int(g.integers(1, 9))
        # one Tc per level's three tables, as the reference's callers build them
        Tc = int(g.choice([1, T]))
        levels.append(tuple(_coeffs(g, mode, Tc, R, n, kind) for _ in range(3)))
    if T0 == 1 and all(lv[0].shape[0] == 1 for lv in levels):
        T = 1
    a, b = _operand(g, mode, T0, N), _operand(g, mode, T0, N)
    return mode, levels, a, b, T


@pytest.mark.parametrize("seed", range(60))
def test_apply_levels_random_problem_bitwise(eng, monkeypatch, seed):
    mode, levels, a, b, T = _problem(seed)
    monkeypatch.setenv("RBC_DETECT_PLANS", "0")
    try:
        with np.errstate(all="ignore"):
            want = oracle.apply_levels(levels, a, b, mode)
    except OverflowError:  # non-finite output: the reference raises (_engine.py:146-148)
        with pytest.raises(OverflowError, match="result left the"):
            eng.apply_levels(levels, a, b, mode)
        return
    stats = {}
    got = eng.apply_levels(levels, a, b, mode, stats)
    assert got.dtype == want.dtype and got.shape == want.shape == (T,) + a.shape[1:]
    assert got.tobytes() == want.tobytes()
    leaves = 1
    for lv in levels:
        leaves *= lv[0].shape[1]
    assert stats["leaf_multiplies"] == T * leaves
    monkeypatch.setenv("RBC_DETECT_PLANS", "1")
    assert same_values(eng.apply_levels(levels, a, b, mode), want)


@pytest.mark.parametrize("seed", range(40))
def test_leaf_matmul_random_shapes_bitwise(eng, seed):
    g = np.random.default_rng(2000 + seed)
    mode = mode_for(LABELS[seed % 3])
    lead = tuple(int(v) for v in g.integers(1, 4, size=int(g.integers(0, 3))))
    M, K, N = (int(v) for v in g.integers(1, 40, size=3))
    if seed % 5 == 0:
        M, K, N = M + 120, K + 60, N + 130  # tiled kernels with ragged edges
    xl = lead if g.random() < 0.7 else (1,) * len(lead)
    yl = lead if g.random() < 0.7 else (1,) * len(lead)
    x = mode.array(g.standard_normal(xl + (M, K)))
    y = mode.array(g.standard_normal(yl + (K, N)))
    x[..., 0, :] = -0.0
    with np.errstate(all="ignore"):
        want = oracle.leaf(np.broadcast_to(x, np.broadcast_shapes(xl, yl) + (M, K)),
                           np.broadcast_to(y, np.broadcast_shapes(xl, yl) + (K, N)))
    got = eng.leaf_matmul(x, y, mode)
    assert got.shape == want.shape and got.dtype == want.dtype
    assert got.tobytes() == want.tobytes()


def _formula(name):
    import paper_1905_07439_b200 as rbc
    from paper_1905_07439_b200.formula import standard_formula

    return {"strassen": rbc.strassen_formula, "laderman": rbc.laderman_formula,
            "standard2": lambda: standard_formula(2), "standard3": lambda: standard_formula(3)}[name]()


def _plan_problem(seed):
    """Exact +-1 formula, random depth / leaf side / trial layout: the plan
    kernels, the two-level passes and whichever fused subtree instantiation
    covers the leaf side."""
    import paper_1905_07439_b200 as rbc

    g = np.random.default_rng(3000 + seed)
    label = LABELS[seed % 3]
    mode = mode_for(label)
    fname = str(g.choice(["strassen", "laderman", "standard2", "standard3"]))
    f = _formula(fname)
    Q = int(g.integers(1, 5 if f.n == 2 else 4))
    m = int(g.choice([1, 2, 3, 4, 5, 8, 9, 10, 16, 27, 32, 35]))
    while m * f.n ** Q > 300:
        m = max(1, m // 2)
    N = m * f.n ** Q
    T = int(g.integers(1, 5))
    T0 = int(g.choice([1, T]))
    a, b = _operand(g, mode, T0, N), _operand(g, mode, T0, N)
    rplans = [rbc.draw_recursive_plan(f.n, Q, rbc.derive_rng(3000 + seed, t)) for t in range(T)]
    return mode, f, Q, a, b, rplans


@pytest.mark.parametrize("seed", range(48))
def test_apply_plans_random_problem_vs_oracle(eng, seed):
    import paper_1905_07439_b200 as rbc
    from paper_1905_07439_b200.randomize import pack_recursive_plans, plan_formula_id

    mode, f, Q, a, b, rplans = _plan_problem(seed)
    packed = pack_recursive_plans(rplans, Q, f.n)
    levels = [rbc.plan_levels(f, [rp.levels[q] for rp in rplans], mode) for q in range(Q)]
    try:
        with np.errstate(all="ignore"):
            want = oracle.apply_levels(levels, a, b, mode)
    except OverflowError:
        with pytest.raises(OverflowError):
            eng.apply_plans(plan_formula_id(f), Q, packed, a, b, mode)
        return
    got = eng.apply_plans(plan_formula_id(f), Q, packed, a, b, mode)
    assert same_values(got, want)


@pytest.mark.parametrize("seed", range(18))
def test_error_trials_random_problem_vs_oracle(seed):
    """The error-trial pipeline (truth, deterministic and randomized products,
    errors, overflow flags) on random small configurations, host buffers."""
    import paper_1905_07439_b200 as rbc
    from paper_1905_07439_b200 import _lib
    from paper_1905_07439_b200.trials import error_trials

    _lib.require_device()
    mode, f, Q, _, _, _ = _plan_problem(seed)
    g = np.random.default_rng(4000 + seed)
    T = int(g.integers(1, 7))
    N = int(g.choice([1, 2, 3, 5, 9])) * f.n ** Q
    if N > 300:
        pytest.skip("size drawn too large for a per-trial oracle check")
    A, B = _operand(g, mode, T, N), _operand(g, mode, T, N)
    rplans = [rbc.draw_recursive_plan(f.n, Q, rbc.derive_rng(4000 + seed, t)) for t in range(T)]
    out = error_trials(f, Q, A, B, mode, rplans=rplans)
    ident = rbc.RecursivePlan(tuple(rbc.identity_plan(f.n) for _ in range(Q)))
    for t in range(T):
        ref = oracle.standard_multiply(A[t].astype(np.float64), B[t].astype(np.float64))
        for key, flag, rp in (("err_rand", "nf_rand", rplans[t]), ("err_det", "nf_det", ident)):
            levels = [rbc.plan_levels(f, [rp.levels[q]], mode) for q in range(Q)]
            try:
                with np.errstate(all="ignore"):
                    C = oracle.apply_levels(levels, A[t:t + 1], B[t:t + 1], mode)
            except OverflowError:
                assert out[flag][t]
                continue
            assert not out[flag][t]
            want = oracle.rel_errors(C, ref)[0]
            assert np.isclose(out[key][t], want, rtol=1e-12, atol=0), (key, t, out[key][t], want)


@pytest.mark.parametrize("seed", range(24))
def test_truth_random_shapes_bitwise(eng, seed):
    """Binary64 truth of mode-typed operands at odd and ragged sizes (register
    tiles below 512, the bulk-copy pipeline above)."""
    g = np.random.default_rng(5000 + seed)
    mode = mode_for(LABELS[seed % 3])
    N = int(g.choice([1, 7, 33, 127, 129, 243, 255, 300, 513, 600]))
    T = int(g.integers(1, 4)) if N < 400 else 1
    A, B = _operand(g, mode, T, N), _operand(g, mode, T, N)
    got = eng.truth(A, B, mode)
    for t in range(T):
        want = oracle.standard_multiply(A[t].astype(np.float64), B[t].astype(np.float64))
        assert got[t].tobytes() == want.tobytes()
