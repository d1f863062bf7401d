"""CPU: the C++ restatement of numpy's SeedSequence / Philox / bounded-integer
/ shuffle algorithms (csrc/hostrng.cu; reference rng.py:20-29 and
randomize.py:118-127) against numpy itself, bit for bit.  Host code only: no
GPU needed, but librbc.so must be built."""

import numpy as np
import pytest

from paper_1905_07439_b200 import hostrng
from paper_1905_07439_b200.randomize import draw_plan
from paper_1905_07439_b200.rng import derive_rng, derive_seed

PATHS = ([(1, p, k) for p in range(1, 60) for k in (0, 1)] + [(2, t, q) for t in (1, 7, 999) for q in range(6)]
         + [(0, 0, 0), (3,), (), (2 ** 32, 5), (2 ** 40 + 3, 2 ** 33, 1, 2, 3), (5, 2 ** 63 + 11)])
SEEDS = [0, 1, 2 ** 31 - 1, 2 ** 32, 12345678901234567, 2 ** 64 - 1]


@pytest.mark.parametrize("seed", SEEDS)
def test_derive_seeds_match_numpy(seed):
    for depth in sorted({len(p) for p in PATHS}):
        paths = [p for p in PATHS if len(p) == depth]
        got = hostrng.derive_seeds(seed, paths)
        assert [int(x) for x in got] == [derive_seed(seed, *p) for p in paths]


@pytest.mark.parametrize("seed", SEEDS)
def test_philox_keys_match_numpy(seed):
    for depth in sorted({len(p) for p in PATHS}):
        paths = [p for p in PATHS if len(p) == depth]
        got = hostrng.philox_keys(seed, paths)
        for k, p in zip(got, paths):
            want = np.random.Philox(np.random.SeedSequence(seed, spawn_key=p)).state["state"]["key"]
            assert (int(k[0]), int(k[1])) == (int(want[0]), int(want[1]))


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8])
def test_draw_plans_match_reference_draw(n):
    paths = [(2, t, q) for t in range(1, 120) for q in range(3)]
    perms, signs = hostrng.draw_plans(n, 1, paths)
    for i, p in enumerate(paths):
        want = draw_plan(n, derive_rng(1, *p))
        assert np.array_equal(perms[i], want.perms) and np.array_equal(signs[i], want.signs), p


def test_stream_words_match_numpy_generator():
    """Plans consume the stream through next_uint32 (two per 64-bit word):
    an odd number of 32-bit draws between plans' rows exercises the half-word
    buffer (n = 3: 9 sign draws, then the shuffles)."""
    paths = [(9, t) for t in range(200)]
    perms, signs = hostrng.draw_plans(3, 77, paths)
    for i, p in enumerate(paths):
        g = derive_rng(77, *p)
        s = 1.0 - 2.0 * g.integers(0, 2, size=(3, 3)).astype(np.float64)
        ps = np.stack([g.permutation(3) for _ in range(3)])
        assert np.array_equal(s, signs[i]) and np.array_equal(ps, perms[i])


def test_per_stream_seeds_match_numpy():
    """One seed per stream (the matrix streams derive_rng(mseed_p, which))."""
    seeds = [derive_seed(1, 1, p, 0) for p in range(1, 40)]
    keys = hostrng.philox_keys(seeds, [(w,) for w in [0, 1] * 19 + [0]])
    for s, w, k in zip(seeds, [0, 1] * 19 + [0], keys):
        want = np.random.Philox(np.random.SeedSequence(s, spawn_key=(w,))).state["state"]["key"]
        assert (int(k[0]), int(k[1])) == (int(want[0]), int(want[1]))


@pytest.mark.parametrize("name", ["c1", "c2", "c4", "c5"])
def test_config_plans_and_pair_seeds(name):
    """The bench's plan records and pair seeds through the native RNG equal
    the numpy-object path (cfg.plan + pack_recursive_plans, derive_seed)."""
    from paper_1905_07439_b200.configs import get_config, packed_plans, pair_seeds
    from paper_1905_07439_b200.matgen import kind_index
    from paper_1905_07439_b200.randomize import pack_recursive_plans

    cfg = get_config(name)
    keys = [cfg.plan_key(p) for p in range(5, 40)]
    want = pack_recursive_plans([cfg.plan(k) for k in keys], cfg.Q, cfg.n)
    assert np.array_equal(packed_plans(cfg, keys), want)
    assert pair_seeds(cfg, 11, 9) == [derive_seed(cfg.seed, 1, p, kind_index(cfg.kind))
                                      for p in range(11, 20)]
