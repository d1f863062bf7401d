"""Seeded substreams, identical to the reference's (``pkg/src/randbc/rng.py:14-36``).

Every random object is drawn on the host from a numpy Philox generator keyed
by ``SeedSequence(seed, spawn_key=path)``, so the plans and inputs this
package uploads to the GPU are the very numbers the reference draws for the
same (seed, path).
"""

from __future__ import annotations

import numpy as np

ROLE_FORMULA = 0
ROLE_MATRIX = 1
ROLE_PLAN = 2
ROLE_INPUT = 3


def _sequence(seed, path) -> np.random.SeedSequence:
    return np.random.SeedSequence(int(seed), spawn_key=tuple(int(p) for p in path))


def derive_rng(seed: int, *path: int) -> np.random.Generator:
    """Philox stream for (seed, *path) (reference rng.py:20-23)."""
    return np.random.Generator(np.random.Philox(_sequence(seed, path)))


def derive_seed(seed: int, *path: int) -> int:
    """u64 master seed derived like derive_rng (reference rng.py:26-29)."""
    return int(_sequence(seed, path).generate_state(1, np.uint64)[0])


def as_generator(rng) -> np.random.Generator:
    if isinstance(rng, np.random.Generator):
        return rng
    return derive_rng(int(rng))
