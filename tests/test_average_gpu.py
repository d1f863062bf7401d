"""GPU: averaging trials (config 3 mechanism: dense noisy-Laderman tables in
binary64, running mean over G plans) against the CPU oracle restating
reference experiments.py:264-296."""

from dataclasses import replace

import numpy as np
import pytest

from oracle import engine as oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,Q,P,G", [(27, 2, 2, 12), (81, 3, 1, 5)])
def test_average_trials_match_oracle(N, Q, P, G):
    from paper_1905_07439_b200.configs import get_config, make_pairs
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.randomize import plan_levels
    from paper_1905_07439_b200.trials import average_trials, checkpoint_grid

    cfg = replace(get_config("c3"), N=N, Q=Q, plans_per_pair=G)
    f = cfg.formula_obj()
    A, B = make_pairs(cfg, 1, P)
    rplans = [cfg.plan(cfg.plan_key(p, j)) for p in range(1, P + 1) for j in range(1, G + 1)]
    got = average_trials(f, Q, A, B, cfg.mode, rplans, G)
    cps = checkpoint_grid(G)
    assert got["checkpoints"] == cps
    for p in range(P):
        ref = oracle.standard_multiply(A[p], B[p])
        refnorm = float(np.linalg.norm(ref.ravel()))
        det = oracle.apply_levels([mode_tensors(f, cfg.mode)] * Q, A[p][None], B[p][None], cfg.mode)
        assert got["err_det"][p] == pytest.approx(oracle.rel_errors(det, ref)[0], rel=1e-12)
        mine = rplans[p * G:(p + 1) * G]
        levels = [plan_levels(f, [rp.levels[q] for rp in mine], cfg.mode) for q in range(Q)]
        C = oracle.apply_levels(levels, A[p][None], B[p][None], cfg.mode)
        np.testing.assert_allclose(got["err_rand"][p], oracle.rel_errors(C, ref), rtol=1e-12)
        total = np.zeros(ref.shape)
        want = []
        for t in range(G):
            np.add(total, C[t], out=total)
            if t + 1 in cps:
                want.append(float(np.linalg.norm((total / (t + 1) - ref).ravel())) / refnorm)
        np.testing.assert_allclose(got["err_mean"][p], want, rtol=1e-12)


def test_average_set_pipelined_equals_serial_and_host_call():
    """trials.run_average_set (fresh pairs drawn on the GPU, plans drawn
    natively, dense tables hatted on the host; the next pass prepared while a
    pass computes) equals its unpipelined run bitwise and the host-buffer
    average_trials call on host-drawn pairs (ragged last pass)."""
    from dataclasses import replace

    from paper_1905_07439_b200.configs import get_config, make_pairs
    from paper_1905_07439_b200.trials import average_trials, run_average_set

    cfg = replace(get_config("c3"), N=81, Q=2, plans_per_pair=5)
    total, P_step = 7, 3
    a = run_average_set(cfg, 2, total, P_step, "cuda:0", pipelined=True)
    b = run_average_set(cfg, 2, total, P_step, "cuda:0", pipelined=False)
    for k in ("err_rand", "err_mean", "err_det"):
        assert a[k].tobytes() == b[k].tobytes(), k
    A, B = make_pairs(cfg, 2, total)
    rplans = [cfg.plan(cfg.plan_key(p, j)) for p in range(2, 2 + total) for j in range(1, 6)]
    host = average_trials(cfg.formula_obj(), cfg.Q, A, B, cfg.mode, rplans, 5)
    for k in ("err_rand", "err_mean", "err_det"):
        assert np.array_equal(a[k], host[k]), k
