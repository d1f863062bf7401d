"""GPU parity: the B200 engine (through the C ABI) against the reference's
golden outputs and the CPU oracle on the same seeded inputs."""

import numpy as np
import pytest

from conftest import case_levels, mode_for, same_values
from oracle import engine as oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    from paper_1905_07439_b200 import _lib, engine

    _lib.require_device()
    return engine


@pytest.mark.parametrize("detect", ["0", "1"])
def test_golden_engine_cases_dense_path(eng, engine_cases, monkeypatch, detect):
    """apply_levels == reference, with hatted +-1 tables recognised and run
    on the plan kernels (detect=1) and with everything dense (detect=0)."""
    monkeypatch.setenv("RBC_DETECT_PLANS", detect)
    meta, arrs = engine_cases
    for case in meta["engine"]:
        name = case["name"]
        mode = mode_for(case["mode"])
        levels = case_levels(arrs, name, case["Q"])
        a, b = arrs[f"{name}/a"], arrs[f"{name}/b"]
        stats = {}
        if case["raises"] == "OverflowError":
            with pytest.raises(OverflowError, match="result left the half range"):
                eng.apply_levels(levels, a, b, mode, stats)
            continue
        out = eng.apply_levels(levels, a, b, mode, stats)
        assert same_values(out, arrs[f"{name}/out"]), name
        assert stats["leaf_multiplies"] == case["leaf_multiplies"], name


def test_golden_engine_cases_plan_path(eng, engine_cases):
    """apply_plans (plans folded into generated networks) == reference."""
    from paper_1905_07439_b200._lib import FORMULA_IDS

    meta, arrs = engine_cases
    checked = 0
    for case in meta["engine"]:
        if case["plan_formula"] is None or f"{case['name']}/perms" not in arrs:
            continue
        name = case["name"]
        mode = mode_for(case["mode"])
        Q, n = case["Q"], case["n"]
        perms, signs = arrs[f"{name}/perms"], arrs[f"{name}/signs"]
        Tp = perms.shape[0]
        packed = eng.pack_plans(n, perms.reshape(Tp * Q, 3, n), signs.reshape(Tp * Q, 3, n))
        packed = packed.reshape(Tp, Q, -1)
        a, b = arrs[f"{name}/a"], arrs[f"{name}/b"]
        fid = FORMULA_IDS[case["plan_formula"]]
        if case["raises"] == "OverflowError":
            with pytest.raises(OverflowError):
                eng.apply_plans(fid, Q, packed, a, b, mode)
            out, flags = eng.apply_plans(fid, Q, packed, a, b, mode, return_flags=True)
            assert flags.all()
            continue
        stats = {}
        out = eng.apply_plans(fid, Q, packed, a, b, mode, stats)
        assert same_values(out, arrs[f"{name}/out"]), name
        assert stats["leaf_multiplies"] == case["leaf_multiplies"], name
        checked += 1
    assert checked >= 8


def test_golden_leaf_cases(eng, engine_cases):
    meta, arrs = engine_cases
    for case in meta["leaf"]:
        name = case["name"]
        mode = mode_for(case["mode"])
        out = eng.leaf_matmul(arrs[f"{name}/x"], arrs[f"{name}/y"], mode)
        assert same_values(out, arrs[f"{name}/out"]), name


@pytest.mark.parametrize(
    "label,fname,Q,N,T",
    [
        ("f32", "strassen", 2, 256, 3),   # config-1 shape
        ("f32", "strassen", 3, 320, 2),   # golden artifact size
        ("f32", "laderman", 3, 81, 3),
        ("f64", "laderman", 2, 81, 2),
        ("f16", "strassen", 3, 128, 2),
        ("f16", "strassen", 1, 256, 2),   # 128x128 half2 tiled leaves
        ("f16", "strassen", 2, 280, 1),   # 70x70 leaves, half2 64-tile with edges
        ("f64", "strassen", 2, 200, 2),
        ("f64", "strassen", 1, 260, 1),   # 130x130 binary64 leaves
    ],
)
def test_random_plans_vs_oracle(eng, monkeypatch, label, fname, Q, N, T):
    """Every engine path equals the oracle on seeded larger problems."""
    import paper_1905_07439_b200 as rbc

    mode = mode_for(label)
    f = {"strassen": rbc.strassen_formula, "laderman": rbc.laderman_formula}[fname]()
    g = rbc.derive_rng(77, N, Q)
    A = mode.array(g.standard_normal((N, N)))
    B = mode.array(g.standard_normal((N, N)))
    rplans = [rbc.draw_recursive_plan(f.n, Q, rbc.derive_rng(78, t)) for t in range(T)]
    levels = [rbc.plan_levels(f, [rp.levels[q] for rp in rplans], mode) for q in range(Q)]
    want = oracle.apply_levels(levels, A[None], B[None], mode)
    got_detected = eng.apply_levels(levels, A[None], B[None], mode)
    got_plan = rbc.recursive_randomized_apply_many(f, rplans, A, B, mode)
    monkeypatch.setenv("RBC_DETECT_PLANS", "0")
    got_dense = eng.apply_levels(levels, A[None], B[None], mode)
    assert same_values(got_dense, want)
    assert same_values(got_detected, want)
    assert same_values(got_plan, want)


@pytest.mark.parametrize(
    "label,fname,Q,N,T,T0",
    [
        ("f32", "laderman", 4, 243, 2, 2),   # config-2 shape: fused bottom 2 levels, 3x3 leaves
        ("f32", "strassen", 5, 320, 2, 1),   # golden artifact shape: 10x10 leaves
        ("f32", "laderman", 2, 9, 3, 3),     # whole recursion fused (q0 = 0), per-trial operands
        ("f64", "laderman", 2, 27, 2, 1),
        ("f16", "laderman", 2, 27, 2, 2),
        ("f16", "strassen", 3, 32, 3, 1),
    ],
)
def test_fused_subtree_vs_breadth_first_and_oracle(eng, monkeypatch, label, fname, Q, N, T, T0):
    import paper_1905_07439_b200 as rbc
    from paper_1905_07439_b200.randomize import pack_recursive_plans, plan_formula_id

    mode = mode_for(label)
    f = {"strassen": rbc.strassen_formula, "laderman": rbc.laderman_formula}[fname]()
    g = rbc.derive_rng(91, N, Q)
    a = mode.array(g.standard_normal((T0, N, N)))
    b = mode.array(g.standard_normal((T0, N, N)))
    rplans = [rbc.draw_recursive_plan(f.n, Q, rbc.derive_rng(92, t)) for t in range(T)]
    packed = pack_recursive_plans(rplans, Q, f.n)
    fid = plan_formula_id(f)
    fused = eng.apply_plans(fid, Q, packed, a, b, mode)
    monkeypatch.setenv("RBC_NO_FUSION", "1")
    plain = eng.apply_plans(fid, Q, packed, a, b, mode)
    monkeypatch.delenv("RBC_NO_FUSION")
    levels = [rbc.plan_levels(f, [rp.levels[q] for rp in rplans], mode) for q in range(Q)]
    want = oracle.apply_levels(levels, a, b, mode)
    assert same_values(plain, want)
    assert same_values(fused, want)


@pytest.mark.parametrize(
    "label,fname,Q,N,T,T0",
    [
        ("f32", "laderman", 3, 243, 2, 2),   # expand2 (levels 0-1) then the fused subtree
        ("f32", "laderman", 4, 243, 2, 2),   # config 2's schedule at two trials
        ("f32", "strassen", 5, 512, 2, 1),   # expand2 twice, then one single level
        ("f16", "strassen", 4, 256, 2, 2),
        ("f64", "strassen", 3, 96, 3, 1),
        ("f64", "laderman", 3, 81, 2, 2),    # no binary64 n=3 instantiation: single levels
    ],
)
@pytest.mark.parametrize("fusion", ["1", "0"])
def test_two_level_expansion_vs_single_levels(eng, monkeypatch, label, fname, Q, N, T, T0, fusion):
    """expand2_plan_kernel / contract2_plan_kernel (two expansion and two
    contraction levels per pass) equal the one-level-per-pass schedule and the
    oracle, with and without the fused bottom subtree (the contraction pairs
    then start at different levels)."""
    import paper_1905_07439_b200 as rbc
    from paper_1905_07439_b200.randomize import pack_recursive_plans, plan_formula_id

    mode = mode_for(label)
    f = {"strassen": rbc.strassen_formula, "laderman": rbc.laderman_formula}[fname]()
    g = rbc.derive_rng(93, N, Q)
    a = mode.array(g.standard_normal((T0, N, N)))
    b = mode.array(g.standard_normal((T0, N, N)))
    rplans = [rbc.draw_recursive_plan(f.n, Q, rbc.derive_rng(94, t)) for t in range(T)]
    packed = pack_recursive_plans(rplans, Q, f.n)
    fid = plan_formula_id(f)
    if fusion == "0":
        monkeypatch.setenv("RBC_NO_FUSION", "1")
    two = eng.apply_plans(fid, Q, packed, a, b, mode)
    monkeypatch.setenv("RBC_NO_EXPAND2", "1")
    one = eng.apply_plans(fid, Q, packed, a, b, mode)
    levels = [rbc.plan_levels(f, [rp.levels[q] for rp in rplans], mode) for q in range(Q)]
    want = oracle.apply_levels(levels, a, b, mode)
    assert one.tobytes() == two.tobytes()
    assert same_values(two, want)


def test_fused_overflow_flags(eng):
    """fp16 overflow inside a fused subtree is flagged per trial."""
    import paper_1905_07439_b200 as rbc
    from paper_1905_07439_b200.randomize import pack_recursive_plans

    mode = mode_for("f16")
    f = rbc.laderman_formula()
    g = rbc.derive_rng(93)
    a = g.standard_normal((2, 27, 27))
    b = g.standard_normal((2, 27, 27))
    a[1] *= 300.0
    b[1] *= 300.0
    a, b = mode.array(a), mode.array(b)
    rplans = [rbc.draw_recursive_plan(3, 2, rbc.derive_rng(94, t)) for t in range(2)]
    packed = pack_recursive_plans(rplans, 2, 3)
    out, flags = eng.apply_plans(2, 2, packed, a, b, mode, return_flags=True)
    assert flags.tolist() == [False, True]
    with pytest.raises(OverflowError):
        eng.apply_plans(2, 2, packed, a, b, mode)


def test_dense_formula_tree_order(eng):
    """Dense (noisy Laderman) coefficients exercise the row-then-rows fold."""
    import paper_1905_07439_b200 as rbc

    mode = mode_for("f32")
    f = rbc.perturb_all(rbc.laderman_formula(), 1e-4, rbc.derive_rng(5, 0))
    g = rbc.derive_rng(6)
    A = mode.array(g.standard_normal((54, 54)))
    B = mode.array(g.standard_normal((54, 54)))
    rplans = [rbc.draw_recursive_plan(3, 2, rbc.derive_rng(7, t)) for t in range(3)]
    levels = [rbc.plan_levels(f, [rp.levels[q] for rp in rplans], mode) for q in range(2)]
    want = oracle.apply_levels(levels, A[None], B[None], mode)
    assert same_values(rbc.recursive_randomized_apply_many(f, rplans, A, B, mode), want)


def test_engine_errors(eng):
    from paper_1905_07439_b200.precision import SINGLE

    one = np.ones((1, 4, 4), np.float32)
    with pytest.raises(ValueError, match="need at least one level"):
        eng.apply_levels([], one, one, SINGLE)
    u = np.ones((1, 7, 3, 3), np.float32)
    with pytest.raises(ValueError, match="not divisible"):
        eng.apply_levels([(u, u, u)], one, one, SINGLE)
    with pytest.raises(ValueError, match="inner dimensions"):
        eng.leaf_matmul(np.ones((1, 2, 3)), np.ones((1, 2, 3)), SINGLE)

    class Dec:
        kind = "decimal"

    with pytest.raises(NotImplementedError):
        eng.apply_levels([(u, u, u)], one, one, Dec())


@pytest.mark.parametrize("detect", ["0", "1"])
def test_empty_operands_after_nonempty_call(eng, monkeypatch, detect):
    """(T, 0, 0) operands return an empty (T, 0, 0) array like the reference,
    also right after a non-empty call left operand bytes in the arena where
    the overflow flags of the empty call land (engine.cu run_pass)."""
    from paper_1905_07439_b200 import SINGLE, strassen_formula
    from paper_1905_07439_b200.multiply import mode_tensors

    monkeypatch.setenv("RBC_DETECT_PLANS", detect)
    f = strassen_formula()
    levels = [mode_tensors(f, SINGLE)] * 2
    rng = np.random.default_rng(5)
    # non-empty call whose operands are far from zero bytes
    a = np.full((1, 64, 64), 3.0e38, np.float32) * rng.choice([-1, 1], (1, 64, 64)).astype(np.float32)
    b = np.ones((1, 64, 64), np.float32)
    with pytest.raises(OverflowError):
        eng.apply_levels(levels, a, b, SINGLE)
    for T in (1, 3):
        e = np.zeros((T, 0, 0), np.float32)
        out = eng.apply_levels(levels, e, e, SINGLE)
        assert out.shape == (T, 0, 0) and out.dtype == np.float32

