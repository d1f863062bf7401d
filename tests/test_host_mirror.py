"""Host-side mirror of the reference's L0/L2 objects, pinned against values
produced by the reference (tests/golden/host_cases.npz).  CPU only."""

import numpy as np
import pytest

import paper_1905_07439_b200 as rbc


def test_draw_plan_matches_reference(host_cases):
    for seed in range(4):
        for n in (2, 3):
            p = rbc.draw_plan(n, rbc.derive_rng(seed, 2, seed + 1, n))
            assert np.array_equal(p.signs, host_cases[f"plan/{seed}/{n}/signs"])
            assert np.array_equal(p.perms, host_cases[f"plan/{seed}/{n}/perms"])


def test_perturb_kappa_hatted(host_cases):
    f = rbc.perturb(rbc.strassen_formula(), 1e-3, 5, rbc.derive_rng(42))
    for x in "uvw":
        assert np.array_equal(getattr(f, x), host_cases[f"perturbed/{x}"])
    assert rbc.kappa(f) == float(host_cases["perturbed/kappa"])
    plan = rbc.RandomizationPlan(host_cases["hatted/signs"], host_cases["hatted/perms"])
    for x, t in zip("uvw", rbc.hatted_tensors(f, plan)):
        assert np.array_equal(t, host_cases[f"hatted/{x}"])


def test_laderman_noisy_kappa(host_cases):
    f = rbc.perturb_all(rbc.laderman_formula(), 1e-4, rbc.derive_rng(1, 0))
    assert rbc.kappa(f) == float(host_cases["laderman_noisy/kappa"])


def test_matgen_and_seeds(host_cases):
    seed = rbc.derive_seed(1, 1, 0, 0)
    assert seed == int(host_cases["derive_seed/1_1_0_0"])
    for kind in ("gaussian", "uniform", "adv1", "adv2", "adv3", "hilbert"):
        A, B = rbc.generate(rbc.MatrixSpec(kind, 6, seed))
        assert np.array_equal(A, host_cases[f"matgen/{kind}/A"]), kind
        assert np.array_equal(B, host_cases[f"matgen/{kind}/B"]), kind


def test_formulas_exact_and_file_format(tmp_path):
    for f in (rbc.strassen_formula(), rbc.laderman_formula(), rbc.standard_formula(3)):
        assert rbc.is_exact(f) and rbc.kappa(f) == 0.0
        p = tmp_path / "f.txt"
        rbc.save_formula(f, p)
        g = rbc.load_formula(p)
        assert all(np.array_equal(getattr(f, x), getattr(g, x)) for x in "uvw")
    with pytest.raises(ValueError):
        rbc.parse_formula("nope")


def test_modes_and_validation():
    assert rbc.SINGLE.array([1.5]).dtype == np.float32
    assert rbc.HALF.array([1.5]).dtype == np.float16
    with pytest.raises(OverflowError):
        rbc.HALF.array([1e6])
    with pytest.raises(ValueError):
        rbc.SINGLE.array([np.inf])
    with pytest.raises(ValueError):
        rbc.RandomizationPlan(np.ones((3, 2)) * 0.5, np.tile(np.arange(2), (3, 1)))
    with pytest.raises(ValueError):
        rbc.RecursivePlan(())
    from paper_1905_07439_b200.precision import mode_of

    class Dec:
        kind = "decimal"

    with pytest.raises(NotImplementedError):
        mode_of(Dec())


def test_config_seed_layout_matches_experiments():
    """Config pairs / plans follow experiments.py:237-245 (pair = repeat index
    in the matrix path; plan stream (seed, ROLE_PLAN, trial, level))."""
    from paper_1905_07439_b200.configs import get_config

    cfg = get_config("c1")
    A, B = cfg.pair(3)
    A64, B64 = rbc.generate(rbc.MatrixSpec("gaussian", 256, rbc.derive_seed(1, 1, 3, 0)))
    assert np.array_equal(A, rbc.SINGLE.array(A64)) and np.array_equal(B, rbc.SINGLE.array(B64))
    rp = cfg.plan(cfg.plan_key(3))
    p0 = rbc.draw_plan(2, rbc.derive_rng(1, 2, 3, 0))
    assert np.array_equal(rp.levels[0].perms, p0.perms)
    c3 = get_config("c3")
    assert c3.plan_key(2, 5) == 37


@pytest.mark.parametrize("name", ["strassen", "laderman", "standard2", "standard3"])
def test_plan_recognition_reproduces_tables(name):
    """engine.match_plans recovers plans whose hatted tables equal the ones
    the reference's L2 builds (randomize.py:163-178), so the drop-in boundary
    can route them to the plan-path kernels."""
    from paper_1905_07439_b200.engine import match_plans
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.randomize import plan_levels

    f = {"strassen": rbc.strassen_formula, "laderman": rbc.laderman_formula,
         "standard2": lambda: rbc.standard_formula(2),
         "standard3": lambda: rbc.standard_formula(3)}[name]()
    Q, T = 2, 40
    rps = [[rbc.draw_plan(f.n, rbc.derive_rng(7, t, q)) for q in range(Q)] for t in range(T)]
    for mode in (rbc.DOUBLE, rbc.SINGLE, rbc.HALF):
        tabs = [list(plan_levels(f, [rp[q] for rp in rps], mode)) for q in range(Q)]
        fid, perms, signs = match_plans(tabs)
        for t in range(T):
            for q in range(Q):
                plan = rbc.RandomizationPlan(signs=signs[t, q], perms=perms[t, q])
                got = plan_levels(f, [plan], mode)
                for a, b in zip(got, tabs[q]):
                    np.testing.assert_array_equal(a[0], b[t])
        # a broadcast (Tc == 1) deterministic level mixes with per-trial ones
        mixed = [list(mode_tensors(f, mode))] + tabs[1:]
        fid2, perms2, _ = match_plans(mixed)
        assert fid2 == fid and perms2.shape == (T, Q, 3, f.n)
        assert np.array_equal(perms2[:, 0], np.tile(np.arange(f.n), (T, 3, 1)))
    # perturbed (non +-1) and mixed-formula levels stay on the dense path
    g = rbc.perturb(f, 1e-3, 0, rbc.derive_rng(5))
    assert match_plans([list(mode_tensors(g, rbc.DOUBLE))]) is None
    u, v, w = (t.copy() for t in mode_tensors(f, rbc.DOUBLE))
    u[0, 0, 0, 0] = -u[0, 0, 0, 0] if u[0, 0, 0, 0] else 1.0
    assert match_plans([[u, v, w]]) is None


@pytest.mark.parametrize("n", [1, 2, 3])
def test_all_plan_arrays_follow_enumeration_order(n):
    """The array form of the plan enumeration (randomize.all_plan_arrays)
    equals the reference order of _all_plans (randomize.py:282-290)."""
    from paper_1905_07439_b200.randomize import _all_plans, all_plan_arrays, plan_count

    perms, signs = all_plan_arrays(n)
    plans = list(_all_plans(n))
    assert len(perms) == len(plans) == plan_count(n)
    step = 1 if n < 3 else 97
    for i in range(0, len(plans), step):
        assert np.array_equal(perms[i], plans[i].perms) and np.array_equal(signs[i], plans[i].signs)
    assert np.array_equal(perms[-1], plans[-1].perms) and np.array_equal(signs[-1], plans[-1].signs)
