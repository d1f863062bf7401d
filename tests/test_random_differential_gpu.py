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


@pytest.mark.parametrize("seed", range(24))
def test_rescaled_multiply_random_problem_bitwise(seed):
    """Device-resident diagonal rescaling (csrc/rescale.cu) on random sizes,
    schedules, modes and formulas (exact and perturbed) against the CPU oracle
    of reference rescale.py:36-99."""
    import paper_1905_07439_b200 as rbc
    from oracle import rescale as oracle_rescale
    from paper_1905_07439_b200 import _lib
    from paper_1905_07439_b200.formula import perturb
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.rescale import INSIDE, OUTSIDE, rescaled_multiply

    _lib.require_device()
    g = np.random.default_rng(6000 + seed)
    mode = mode_for(LABELS[seed % 3])
    f = rbc.strassen_formula() if seed % 2 else rbc.laderman_formula()
    if seed % 4 >= 2:
        f = perturb(f, 1e-3, 2, rbc.derive_rng(6000 + seed, 0))
    Q = int(g.integers(0, 4 if f.n == 2 else 3))
    N = int(g.integers(1, 6)) * f.n ** Q
    schedule = tuple(g.choice([OUTSIDE, INSIDE], size=int(g.integers(0, 5))))
    scale = np.exp(g.uniform(-2, 2, size=(N, 1)))
    A = mode.array(g.standard_normal((N, N)) * scale)
    B = mode.array(g.standard_normal((N, N)) * scale.T)
    u, v, w = (t[0] for t in mode_tensors(f, mode))
    try:
        with np.errstate(all="ignore"):
            want = oracle_rescale.rescaled_multiply(A, B, Q, schedule, mode, u, v, w)
    except (OverflowError, ValueError) as exc:
        with pytest.raises(type(exc)):
            rescaled_multiply(A, B, Q, schedule, mode, f)
        return
    got = rescaled_multiply(A, B, Q, schedule, mode, f)
    assert got.dtype == want.dtype and np.array_equal(got, want, equal_nan=True)


@pytest.mark.parametrize("seed", range(30))
def test_device_matgen_random_draws_bitwise(seed):
    """The device generator (Philox4x64-10 + numpy's ziggurat, csrc/matgen.cu)
    on random sizes (odd ones too), families, modes and seeds against the host
    draw through numpy (reference matgen.py:55-97)."""
    from paper_1905_07439_b200 import _lib
    from paper_1905_07439_b200.matgen import BUILDER_KINDS, MATRIX_KINDS, MatrixSpec, generate, generate_device

    _lib.require_device()
    g = np.random.default_rng(7000 + seed)
    mode = mode_for(LABELS[seed % 3])
    kinds = MATRIX_KINDS + BUILDER_KINDS
    kind = kinds[seed % len(kinds)]
    n = int(g.choice([2, 3, 4, 7, 16, 31, 64, 100, 129, 257]))
    if kind == "quadrant100":
        n += n % 2
    seeds = [int(s) for s in g.integers(0, 2 ** 63, size=int(g.integers(1, 5)))]
    try:
        want = [[mode.array(m) for m in generate(MatrixSpec(kind, n, s))] for s in seeds]
    except OverflowError:
        with pytest.raises(OverflowError):
            generate_device(kind, n, seeds, mode)
        return
    A, B = generate_device(kind, n, seeds, mode)
    for i in range(len(seeds)):
        assert A[i].cpu().numpy().tobytes() == np.ascontiguousarray(want[i][0]).tobytes(), (kind, n, i)
        assert B[i].cpu().numpy().tobytes() == np.ascontiguousarray(want[i][1]).tobytes(), (kind, n, i)


@pytest.mark.parametrize("seed", range(8))
def test_average_trials_random_problem_vs_oracle(seed):
    """The averaging pipeline (dense tables, running binary64 mean at the
    reference's checkpoints, experiments.py:264-296) on random small problems."""
    import paper_1905_07439_b200 as rbc
    from paper_1905_07439_b200 import _lib
    from paper_1905_07439_b200.formula import perturb
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.trials import average_trials, checkpoint_grid

    _lib.require_device()
    g = np.random.default_rng(8000 + seed)
    mode = mode_for(LABELS[seed % 2])  # f64 / f32
    base = rbc.strassen_formula() if seed % 2 else rbc.laderman_formula()
    f = perturb(base, 1e-3, 3, rbc.derive_rng(8000 + seed, 0))
    Q = int(g.integers(1, 3))
    N = int(g.integers(1, 4)) * f.n ** Q
    P, G = int(g.integers(1, 4)), int(g.integers(1, 14))
    A, B = _operand(g, mode, P, N), _operand(g, mode, P, N)
    rplans = [rbc.draw_recursive_plan(f.n, Q, rbc.derive_rng(8000 + seed, 1, t)) for t in range(P * G)]
    got = average_trials(f, Q, A, B, mode, rplans, G)
    cps = checkpoint_grid(G)
    for p in range(P):
        ref = oracle.standard_multiply(A[p].astype(np.float64), B[p].astype(np.float64))
        refnorm = float(np.linalg.norm(ref.ravel()))
        det = oracle.apply_levels([mode_tensors(f, mode)] * Q, A[p][None], B[p][None], mode)
        assert np.isclose(got["err_det"][p], oracle.rel_errors(det, ref)[0], rtol=1e-12, atol=0)
        mine = rplans[p * G:(p + 1) * G]
        levels = [rbc.plan_levels(f, [rp.levels[q] for rp in mine], mode) for q in range(Q)]
        C = oracle.apply_levels(levels, A[p][None], B[p][None], mode)
        np.testing.assert_allclose(got["err_rand"][p], oracle.rel_errors(C, ref), rtol=1e-12)
        total = np.zeros(ref.shape)
        want = []
        for t in range(G):
            np.add(total, C[t].astype(np.float64), out=total)
            if t + 1 in cps:
                want.append(float(np.linalg.norm((total / (t + 1) - ref).ravel())) / refnorm)
        np.testing.assert_allclose(got["err_mean"][p], want, rtol=1e-12)
