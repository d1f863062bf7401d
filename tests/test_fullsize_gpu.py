"""GPU parity at the full BASELINE sizes (configurations 2-5).

The north-star correctness target is "every config matches the reference
oracle": combinations bit-exact, products value-equal, per-trial errors and
their distribution within tolerance (reference experiments.py:248-261;
_engine.py:146-148: any non-finite output raises).  Where a whole CPU product
takes minutes (configurations 4 and 5: ~100 s and ~680 s per product), the
top recursion level is checked by decomposition:

    C = contract_w0( P_r ),  P_r = sub-product of branch r over levels 1..Q-1
                                    of X_r = expand_u0(A)_r, Y_r = expand_v0(B)_r

with the top-level expansion and contraction on the CPU oracle, the seven
sub-products on the GPU (branch 0 of the next level also on the CPU oracle),
and the GPU's whole product -- the kernels the bench times -- compared value
for value with the decomposed result.  CPU work runs in a process pool
(oracle only; the product path never calls it).
"""

import concurrent.futures as cf
import multiprocessing as mp
import os

import numpy as np
import pytest

from oracle import engine as oracle

pytestmark = pytest.mark.gpu


def _pool(n):
    workers = max(1, min(n, os.cpu_count() or 1, 16))
    return cf.ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn"))


def _levels(cfg, f, key):
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.randomize import plan_levels

    if key == 0:
        return [mode_tensors(f, cfg.mode)] * cfg.Q
    rp = cfg.plan(key)
    return [plan_levels(f, [rp.levels[q]], cfg.mode) for q in range(cfg.Q)]


def _oracle_trial(args):
    """(config, pair p, plan key or 0 for deterministic) -> (overflowed,
    rel error or NaN), whole product on the CPU oracle."""
    name, p, key = args
    from paper_1905_07439_b200.configs import get_config

    cfg = get_config(name)
    f = cfg.formula_obj()
    A, B = cfg.pair(p)
    with np.errstate(all="ignore"):
        try:
            C = oracle.apply_levels(_levels(cfg, f, key), A[None], B[None], cfg.mode)
        except OverflowError:
            return True, float("nan")
    ref = oracle.standard_multiply(A.astype(np.float64), B.astype(np.float64))
    return False, float(oracle.rel_errors(C, ref)[0])


def _oracle_branch(args):
    """Branch-0 sub-product of levels d..Q-1 on the CPU oracle, with its
    sub-operands: (x0, y0, C or None)."""
    name, p, key, d = args
    from paper_1905_07439_b200.configs import get_config

    cfg = get_config(name)
    f = cfg.formula_obj()
    A, B = cfg.pair(p)
    levels = _levels(cfg, f, key)
    x, y = A[None, None], B[None, None]
    with np.errstate(all="ignore"):
        for q in range(d):
            x = oracle.combine(x, levels[q][0][:, :1])
            y = oracle.combine(y, levels[q][1][:, :1])
        try:
            C = oracle.apply_levels(levels[d:], x[:, 0], y[:, 0], cfg.mode)
        except OverflowError:
            C = None
    return x[:, 0], y[:, 0], C


def _packed(cfg, key):
    from paper_1905_07439_b200.randomize import pack_recursive_plans
    from paper_1905_07439_b200.trials import identity_packed

    if key == 0:
        return identity_packed(cfg.n, cfg.Q)
    return pack_recursive_plans([cfg.plan(key)], cfg.Q, cfg.n)


def _same(x, y):
    x, y = np.asarray(x), np.asarray(y)
    return x.dtype == y.dtype and x.shape == y.shape and bool(np.array_equal(x, y, equal_nan=True))


def _decomposition_check(name, key, p=1, d_branch=2):
    """Whole GPU product == oracle contraction of the GPU's 7 sub-products of
    the oracle's top-level expansion; branch 0 of levels d_branch.. on the CPU
    oracle == the same sub-product on the GPU.  Returns (C_gpu, flag)."""
    from paper_1905_07439_b200 import engine
    from paper_1905_07439_b200.configs import get_config
    from paper_1905_07439_b200.randomize import plan_formula_id

    cfg = get_config(name)
    f = cfg.formula_obj()
    fid = plan_formula_id(f)
    with _pool(1) as ex:
        branch = ex.submit(_oracle_branch, (name, p, key, d_branch))
        A, B = cfg.pair(p)
        levels = _levels(cfg, f, key)
        packed = _packed(cfg, key)
        C_gpu, nf = engine.apply_plans(fid, cfg.Q, packed, A[None], B[None], cfg.mode,
                                       return_flags=True)
        with np.errstate(all="ignore"):
            X = oracle.combine(A[None, None], levels[0][0])
            Y = oracle.combine(B[None, None], levels[0][1])
            sub = np.ascontiguousarray(packed[:, 1:])
            P = np.stack([engine.apply_plans(fid, cfg.Q - 1, sub, X[:, r], Y[:, r], cfg.mode,
                                             return_flags=True)[0][0] for r in range(cfg.rank)])
            C_dec = oracle.accumulate(P[None, None], levels[0][2])[:, 0]
        finite = bool(np.all(np.isfinite(C_dec)))
        assert bool(nf[0]) == (not finite), f"{name}: overflow flag"
        # An overflowed product raises in the reference (_engine.py:146-148),
        # so only its flag is observable: the dense reference multiplies every
        # coefficient, zeros included, and 0 * inf spreads NaN into blocks
        # the +-1 plan kernels never touch.
        if finite:
            assert _same(C_gpu, C_dec), f"{name}: whole product differs from the decomposition"
        x0, y0, C0 = branch.result()
    subd = np.ascontiguousarray(packed[:, d_branch:])
    G0, g_nf = engine.apply_plans(fid, cfg.Q - d_branch, subd, x0, y0, cfg.mode, return_flags=True)
    if C0 is None:
        assert g_nf[0], f"{name}: CPU branch overflowed, GPU branch did not"
        assert not np.all(np.isfinite(G0))
    else:
        assert not g_nf[0] and _same(G0, C0), f"{name}: branch-0 sub-product differs"
    return C_gpu, bool(nf[0]), A, B


def test_c5_fullsize_randomized_product_and_error():
    """Configuration 5 (Strassen Q=5, n=8192, f32): pair 1's randomized product
    (plans of trial 1) by decomposition, branch 0 of levels 2..4 (2048^2) on
    the CPU oracle, and the bench path's per-trial error (DeviceErrorTrials)
    against the decomposed product and the binary64 truth."""
    import torch

    from paper_1905_07439_b200 import engine
    from paper_1905_07439_b200.configs import get_config
    from paper_1905_07439_b200.trials import DeviceErrorTrials

    cfg = get_config("c5")
    C, nf, A, B = _decomposition_check("c5", cfg.plan_key(1))
    assert not nf
    ref = engine.truth(A[None], B[None], cfg.mode)[0]
    want = oracle.rel_errors(C, ref)[0]
    runner = DeviceErrorTrials(cfg.formula_obj(), cfg.Q, cfg.N, cfg.mode, 1)
    a = torch.from_numpy(A[None]).cuda()
    b = torch.from_numpy(B[None]).cuda()
    pl = torch.from_numpy(_packed(cfg, cfg.plan_key(1))).cuda()
    runner.run(a, b, pl)
    got = runner.err_rand.cpu().numpy()[0]
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=0)
    assert 1e-6 < got < 1e-4  # f32 Strassen Q=5 anchor ~1e-5


@pytest.mark.parametrize("key", ["det", "rand"])
def test_c4_fullsize_products(key):
    """Configuration 4 (Strassen Q=4, n=2048, binary16, quadrant x100 inputs):
    pair 1's deterministic and randomized products by decomposition (values,
    NaN/inf positions and the overflow flag), branch 0 of levels 1..3
    (1024^2) on the CPU oracle."""
    from paper_1905_07439_b200.configs import get_config

    cfg = get_config("c4")
    _decomposition_check("c4", 0 if key == "det" else cfg.plan_key(1), d_branch=1)


def test_c4_overflow_flags_and_errors_8_pairs():
    """Configuration 4: per-trial overflow flags (and errors of finite trials)
    of 8 pairs, deterministic and randomized, from the error-trial pipeline
    the bench times, against whole CPU-oracle products (one pair per call)."""
    from paper_1905_07439_b200.configs import get_config, make_pairs
    from paper_1905_07439_b200.trials import error_trials

    cfg = get_config("c4")
    T = 8
    jobs = [("c4", p, k) for p in range(1, T + 1) for k in (0, cfg.plan_key(p))]
    with _pool(len(jobs)) as ex:
        fut = ex.map(_oracle_trial, jobs)
        A, B = make_pairs(cfg, 1, T)
        rplans = [cfg.plan(cfg.plan_key(p)) for p in range(1, T + 1)]
        got = error_trials(cfg.formula_obj(), cfg.Q, A, B, cfg.mode, rplans=rplans)
        res = list(fut)
    want_nf = np.array([r[0] for r in res]).reshape(T, 2)
    want_err = np.array([r[1] for r in res]).reshape(T, 2)
    assert np.array_equal(got["nf_det"], want_nf[:, 0])
    assert np.array_equal(got["nf_rand"], want_nf[:, 1])
    for col, k in ((0, "err_det"), (1, "err_rand")):
        ok = ~want_nf[:, col]
        np.testing.assert_allclose(got[k][ok], want_err[ok, col], rtol=1e-12, atol=0)


def test_c3_fullsize_products_errors_and_running_mean():
    """Configuration 3 (noisy Laderman Q=3, n=729, binary64): pair 1's
    deterministic product and plans 1-2 through the drop-in (dense kernels)
    value-equal to the CPU oracle, and the averaging pipeline the bench times
    (DeviceAverageTrials): per-plan, deterministic and running-mean errors at
    1e-12 (reference experiments.py:264-296)."""
    import torch

    from paper_1905_07439_b200 import engine
    from paper_1905_07439_b200.configs import get_config
    from paper_1905_07439_b200.trials import DeviceAverageTrials

    cfg = get_config("c3")
    f = cfg.formula_obj()
    A, B = cfg.pair(1)
    keys = [0, cfg.plan_key(1, 1), cfg.plan_key(1, 2)]
    outs = []
    for key in keys:
        levels = _levels(cfg, f, key)
        got = engine.apply_levels(levels, A[None], B[None], cfg.mode)
        want = oracle.apply_levels(levels, A[None], B[None], cfg.mode)
        assert _same(got, want), f"c3 product key {key}"
        outs.append(want[0])
    ref = oracle.standard_multiply(A, B)
    assert _same(engine.truth(A[None], B[None], cfg.mode)[0], ref)
    errs = [oracle.rel_errors(C[None], ref)[0] for C in outs]
    mean2 = (outs[1] + outs[2]) / 2.0  # total_2 = fl(C1 + C2), mean = fl(total_2 / 2)
    err_mean = [errs[1], oracle.rel_errors(mean2[None], ref)[0]]
    runner = DeviceAverageTrials(f, cfg.Q, cfg.N, cfg.mode, 1, 2, checkpoints=[1, 2])
    tables = runner.tables([cfg.plan(k) for k in keys[1:]])
    runner.run(torch.from_numpy(A[None]).cuda(), torch.from_numpy(B[None]).cuda(), tables)
    torch.cuda.synchronize()
    r = runner.results()
    np.testing.assert_allclose(r["err_det"][0], errs[0], rtol=1e-12, atol=0)
    np.testing.assert_allclose(r["err_rand"][0], errs[1:], rtol=1e-12, atol=0)
    np.testing.assert_allclose(r["err_mean"][0], err_mean, rtol=1e-12, atol=0)


def test_c2_error_distribution_200_pairs():
    """Configuration 2 (Laderman Q=4, n=243, f32, Uniform[-1,1]): 200 pairs'
    per-trial errors, randomized and deterministic, from the error-trial
    pipeline the bench times, against whole CPU-oracle products, and the
    distribution statistics (mean, std, quantiles) reported in the bench line."""
    from paper_1905_07439_b200.configs import get_config, make_pairs
    from paper_1905_07439_b200.distributed import trial_stats
    from paper_1905_07439_b200.trials import error_trials

    cfg = get_config("c2")
    T = 200
    jobs = [("c2", p, k) for p in range(1, T + 1) for k in (0, cfg.plan_key(p))]
    with _pool(len(jobs)) as ex:
        fut = ex.map(_oracle_trial, jobs, chunksize=8)
        A, B = make_pairs(cfg, 1, T)
        rplans = [cfg.plan(cfg.plan_key(p)) for p in range(1, T + 1)]
        got = error_trials(cfg.formula_obj(), cfg.Q, A, B, cfg.mode, rplans=rplans)
        res = list(fut)
    want = np.array([r[1] for r in res]).reshape(T, 2)
    assert not any(r[0] for r in res)
    np.testing.assert_allclose(got["err_det"], want[:, 0], rtol=1e-12, atol=0)
    np.testing.assert_allclose(got["err_rand"], want[:, 1], rtol=1e-12, atol=0)
    gs = trial_stats(got["err_rand"], got["err_det"])
    ws = trial_stats(want[:, 1], want[:, 0])
    for side in ("rand", "det"):
        for stat in ("mean", "std", "q05", "median", "q95"):
            np.testing.assert_allclose(gs[side][stat], ws[side][stat], rtol=1e-10, atol=0)
