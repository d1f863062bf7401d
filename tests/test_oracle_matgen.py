"""CPU: the restatement of the device matrix generator (oracle/matgen.py) is
pinned against numpy's own Philox / Generator, the reference's generator."""

import numpy as np
import pytest

from oracle import matgen as om
from paper_1905_07439_b200.matgen import philox_key


@pytest.mark.parametrize("seed,path", [(1, (0,)), (2**64 - 1, (1,)), (12345, (1, 7, 0))])
def test_philox_stream(seed, path):
    key = philox_key(seed, *path)
    want = np.random.Philox(np.random.SeedSequence(seed, spawn_key=path)).random_raw(37)
    assert om.raw_words(key, 37) == [int(w) for w in want]


def test_random_doubles():
    key = philox_key(9, 0)
    g = np.random.Generator(np.random.Philox(np.random.SeedSequence(9, spawn_key=(0,))))
    want = g.random(64)
    got = np.array([om.unit_double(w) for w in om.raw_words(key, 64)])
    assert got.tobytes() == want.tobytes()


def test_ziggurat_tables_are_numpys():
    ki, wi, fi = om.tables()
    assert len(ki) == len(wi) == len(fi) == 256
    assert fi[0] == 1.0 and ki[1] == 0
    assert abs(wi[255] * 2.0**52 - om.ZIG_R) < 1e-12


@pytest.mark.parametrize("seed", [1, 77])
def test_standard_normal_restatement(seed):
    """60K samples: ~700 wedge tests and ~15 tail samples per stream."""
    n = 60_000
    g = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed, spawn_key=(1,))))
    want = g.standard_normal(n)
    words = om.raw_words(philox_key(seed, 1), int(n * 1.05) + 64)
    got = om.standard_normals(words, n)
    assert got.tobytes() == want.tobytes()
