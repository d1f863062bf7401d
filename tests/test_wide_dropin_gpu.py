"""engine.install(wide=True): the reference's run_experiment with its L2 entry
points (recursive_randomized_apply[_many], recursive_apply, rescaled_multiply)
and experiments._rel_errors routed to this package -- plans, scalings and
error reductions behind the C ABI -- must give the records of the unmodified
reference (run on the CPU here, small sizes) and of the narrow drop-in."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "randbc").is_dir(), reason="baseline/_ref not installed")]


@pytest.fixture()
def randbc():
    from paper_1905_07439_b200 import _lib

    _lib.require_device()
    sys.path.insert(0, str(REF))
    try:
        import randbc
        import randbc.experiments  # noqa: F401
        yield randbc
    finally:
        sys.path.remove(str(REF))


def _records(randbc, experiment, **kw):
    from randbc.experiments import ExperimentConfig, run_experiment
    from randbc.precision import SINGLE

    kw.setdefault("precision", SINGLE)
    kw.setdefault("matrix_type", "gaussian" if experiment.endswith("_avg") else "all")
    cfg = ExperimentConfig(experiment=experiment, seed=3, **kw)
    return run_experiment(cfg)


def _table(records):
    return {(r.experiment, r.algorithm, r.matrix_type, r.n, r.Q, r.trial, r.running_n): r.rel_error
            for r in records}


@pytest.mark.parametrize("experiment,kw", [
    ("s2_variants", dict(size=32, recursions=3, trials=6)),
    ("s2_variants", dict(size=48, recursions=2, trials=5, precision="f64")),
    ("s1_dist", dict(size=32, recursions=2, trials=6)),
    ("s1_avg", dict(size=16, recursions=2, trials=12)),
])
def test_wide_install_reproduces_reference_records(randbc, experiment, kw):
    from randbc.precision import parse_precision

    from paper_1905_07439_b200 import engine

    if "precision" in kw:
        kw = dict(kw, precision=parse_precision(kw["precision"]))
    want = _table(_records(randbc, experiment, **kw))  # unmodified reference, CPU
    engine.install()
    try:
        narrow = _table(_records(randbc, experiment, **kw))
    finally:
        engine.uninstall()
    engine.install(wide=True)
    try:
        import randbc.experiments as rexp

        assert rexp._rel_errors is engine.rel_errors
        wide = _table(_records(randbc, experiment, **kw))
    finally:
        engine.uninstall()
    import randbc.experiments as rexp

    assert rexp._rel_errors is not engine.rel_errors  # restored
    assert want.keys() == narrow.keys() == wide.keys() and len(want) > 10
    for key, w in want.items():
        assert np.isclose(narrow[key], w, rtol=1e-12, atol=0), (key, narrow[key], w)
        assert np.isclose(wide[key], w, rtol=1e-12, atol=0), (key, wide[key], w)


def test_rel_errors_matches_reference_function(randbc):
    from randbc.experiments import _rel_errors
    from randbc.precision import SINGLE

    from paper_1905_07439_b200 import engine

    g = np.random.default_rng(4)
    ref = g.standard_normal((96, 96))
    res = SINGLE.array(ref[None] + 1e-4 * g.standard_normal((7, 96, 96)))
    refnorm = float(np.linalg.norm(ref.ravel()))
    want = _rel_errors(res, ref, refnorm, SINGLE)
    got = engine.rel_errors(res, ref, refnorm, SINGLE)
    assert np.allclose(got, want, rtol=1e-12, atol=0)
