"""The BASELINE.json configurations and their seed layout.

Every input is drawn on the host with the reference's substream layout
(reference experiments.py:237-245, matgen.py:71-72):

* pair p (1-based):  mseed = derive_seed(S, ROLE_MATRIX, p, kind_index)
                     A <- derive_rng(mseed, 0), B <- derive_rng(mseed, 1)
* plan of trial t, level q: draw_plan(n, derive_rng(S, ROLE_PLAN, t, q))
  (config 3: trial key (p - 1) * plans_per_pair + t, so pairs get independent
  plans)
* formula noise (config 3): derive_rng(S, ROLE_FORMULA)

No public dataset is involved: all inputs are seeded synthetic matrices with
the shapes and distributions BASELINE.json names.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .formula import laderman_formula, perturb_all, strassen_formula
from .matgen import MatrixSpec, generate, kind_index
from .precision import DOUBLE, HALF, SINGLE, Mode
from .randomize import RecursivePlan, draw_plan
from .rng import ROLE_FORMULA, ROLE_MATRIX, ROLE_PLAN, derive_rng, derive_seed

__all__ = ["TrialConfig", "CONFIGS", "get_config"]


@dataclass(frozen=True)
class TrialConfig:
    name: str
    formula: str           # strassen | laderman | laderman_noisy
    Q: int
    N: int
    mode: Mode
    kind: str              # matrix family
    trials: int            # operand pairs
    plans_per_pair: int = 1
    seed: int = 1
    note: str = ""

    @property
    def n(self) -> int:
        return 2 if self.formula == "strassen" else 3

    @property
    def rank(self) -> int:
        return 7 if self.formula == "strassen" else 23

    def formula_obj(self):
        if self.formula == "strassen":
            return strassen_formula()
        if self.formula == "laderman":
            return laderman_formula()
        if self.formula == "laderman_noisy":
            return perturb_all(laderman_formula(), 1e-4, derive_rng(self.seed, ROLE_FORMULA))
        raise ValueError(self.formula)

    def pair(self, p: int):
        """Mode-rounded operands of pair p (1-based)."""
        mseed = derive_seed(self.seed, ROLE_MATRIX, p, kind_index(self.kind))
        A, B = generate(MatrixSpec(self.kind, self.N, mseed))
        return self.mode.array(A), self.mode.array(B)

    def plan_key(self, p: int, j: int = 1) -> int:
        return (p - 1) * self.plans_per_pair + j if self.plans_per_pair > 1 else p

    def plan(self, key: int) -> RecursivePlan:
        return RecursivePlan(
            tuple(draw_plan(self.n, derive_rng(self.seed, ROLE_PLAN, key, q)) for q in range(self.Q))
        )

    def effective_flops(self) -> float:
        return 2.0 * float(self.N) ** 3

    def leaf_flops(self) -> float:
        return 2.0 * float(self.N) ** 3 * (self.rank / self.n ** 3) ** self.Q


CONFIGS = {
    "c1": TrialConfig("c1", "strassen", 2, 256, SINGLE, "gaussian", 100,
                      note="Strassen Q=2 n=256 f32, 100 seeded pairs"),
    "c2": TrialConfig("c2", "laderman", 4, 243, SINGLE, "uniform_pm1", 1000,
                      note="Laderman Q=4 n=243 f32 Uniform[-1,1], 1000 pairs, randomized vs deterministic"),
    "c3": TrialConfig("c3", "laderman_noisy", 3, 729, DOUBLE, "gaussian", 500, plans_per_pair=32,
                      note="Laderman+N(0,1e-4) Q=3 n=729 f64, 500 pairs x 32 plans"),
    "c4": TrialConfig("c4", "strassen", 4, 2048, HALF, "quadrant100", 256,
                      note="Strassen Q=4 n=2048 f16, quadrant x100 inputs, 256 pairs"),
    "c5": TrialConfig("c5", "strassen", 5, 8192, SINGLE, "gaussian", 64,
                      note="Strassen Q=5 n=8192 f32, 64 pairs"),
}


def get_config(name: str) -> TrialConfig:
    try:
        return CONFIGS[name]
    except KeyError:
        raise ValueError(f"unknown config {name!r}; choose from {sorted(CONFIGS)}") from None


def pair_seeds(cfg: TrialConfig, first: int, count: int):
    """Matrix seeds mseed of pairs first..first+count-1 (experiments.py:237-239),
    through the native SeedSequence (hostrng; bit-identical to derive_seed)."""
    from . import hostrng

    k = kind_index(cfg.kind)
    return [int(x) for x in hostrng.derive_seeds(
        cfg.seed, [(ROLE_MATRIX, p, k) for p in range(first, first + count)])]


def packed_plans(cfg: TrialConfig, keys) -> np.ndarray:
    """(len(keys), Q, 40) packed plan records of trials ``keys`` (plan of
    trial t, level q: draw_plan(n, derive_rng(S, ROLE_PLAN, t, q))), drawn by
    the native host RNG (hostrng: bit-identical to cfg.plan) and packed for
    the plan kernels."""
    from . import engine, hostrng

    keys = list(keys)
    perms, signs = hostrng.draw_plans(
        cfg.n, cfg.seed, [(ROLE_PLAN, t, q) for t in keys for q in range(cfg.Q)])
    return engine.pack_plans(cfg.n, perms, signs).reshape(len(keys), cfg.Q, -1)


def make_pairs_device(cfg: TrialConfig, first: int, count: int, device="cuda:0", out=None):
    """Device twin of :func:`make_pairs`: (A, B) torch tensors (count, N, N)
    in the mode dtype on ``device``, bit-identical to make_pairs (the matrices
    are drawn on the GPU from the same Philox streams)."""
    from .matgen import generate_device

    return generate_device(cfg.kind, cfg.N, pair_seeds(cfg, first, count), cfg.mode, device,
                           out=out)


def make_pairs(cfg: TrialConfig, first: int, count: int, workers: int = 1):
    """(count, N, N) stacks of pairs first..first+count-1, mode dtype."""
    ids = list(range(first, first + count))
    if workers > 1 and count > 1:
        import concurrent.futures as cf

        with cf.ProcessPoolExecutor(max_workers=workers) as ex:
            pairs = list(ex.map(cfg.pair, ids, chunksize=max(1, count // (4 * workers))))
    else:
        pairs = [cfg.pair(p) for p in ids]
    A = np.stack([pa for pa, _ in pairs])
    B = np.stack([pb for _, pb in pairs])
    return A, B
