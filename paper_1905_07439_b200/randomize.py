"""Random sign/permutation conjugation of bilinear formulas (host side).

Mirror of ``randbc.randomize`` (reference ``pkg/src/randbc/randomize.py``)
with the same names, argument meaning, draw order and errors:

* ``RandomizationPlan`` / ``RecursivePlan``  -- randomize.py:58-110
* ``identity_plan`` / ``draw_plan`` / ``variant_plan`` -- :113-143
* ``hatted_tensors``                         -- :156-178
* ``plan_levels`` (``_plan_levels``)         -- :199-209
* ``randomized_apply`` / ``recursive_randomized_apply[_many]`` -- :212-274

The multiply itself runs on the B200.  For the exact +-1 formulas the
engine has compiled networks for (Strassen, Laderman, standard(2/3)) the
plans are uploaded as-is and folded into the kernels (``engine.apply_plans``);
any other formula goes through hatted coefficient tables and the general
engine (``engine.apply_levels``).  Both give the reference's values.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import engine
from .formula import BilinearFormula, kappa
from .formula import laderman_formula, standard_formula, strassen_formula
from .multiply import _as_operands, _check_blocked
from .precision import DOUBLE, mode_of
from .rng import as_generator

__all__ = [
    "VARIANTS",
    "RandomizationPlan",
    "RecursivePlan",
    "identity_plan",
    "draw_plan",
    "variant_plan",
    "identity_recursive_plan",
    "draw_recursive_plan",
    "hatted_tensors",
    "plan_levels",
    "randomized_apply",
    "recursive_randomized_apply",
    "recursive_randomized_apply_many",
    "plan_formula_id",
    "pack_recursive_plans",
]

VARIANTS = ("full", "sign", "perm", "none")
DEFAULT_CHUNK_ELEMENTS = 1 << 24


@dataclass(frozen=True)
class RandomizationPlan:
    """Signs (3, n) in {-1, +1} and permutations (3, n); perms[i][j] is the
    base block index that block j of the conjugated grid reads."""

    signs: np.ndarray
    perms: np.ndarray

    def __post_init__(self):
        signs = np.array(self.signs, dtype=np.float64)
        perms = np.array(self.perms, dtype=np.int64)
        if signs.ndim != 2 or signs.shape[0] != 3 or signs.shape != perms.shape:
            raise ValueError("signs and perms must both have shape (3, n)")
        if not np.all(np.abs(signs) == 1.0):
            raise ValueError("signs must be +1 or -1")
        want = np.arange(perms.shape[1])
        if any(not np.array_equal(np.sort(row), want) for row in perms):
            raise ValueError("each perms row must be a permutation of 0..n-1")
        signs.flags.writeable = False
        perms.flags.writeable = False
        object.__setattr__(self, "signs", signs)
        object.__setattr__(self, "perms", perms)

    @property
    def n(self) -> int:
        return self.perms.shape[1]


@dataclass(frozen=True)
class RecursivePlan:
    """One plan per recursion level, levels[0] outermost."""

    levels: tuple

    def __post_init__(self):
        levels = tuple(self.levels)
        if not levels:
            raise ValueError("need at least one level")
        if not all(isinstance(p, RandomizationPlan) for p in levels):
            raise ValueError("levels must be RandomizationPlan instances")
        if len({p.n for p in levels}) != 1:
            raise ValueError("levels must share one grid size")
        object.__setattr__(self, "levels", levels)

    @property
    def depth(self) -> int:
        return len(self.levels)

    @property
    def n(self) -> int:
        return self.levels[0].n


def identity_plan(n: int) -> RandomizationPlan:
    return RandomizationPlan(np.ones((3, n)), np.tile(np.arange(n), (3, 1)))


def draw_plan(n: int, rng) -> RandomizationPlan:
    """Uniform plan; draw order: the 3 x n sign grid (row-major), then three
    Fisher-Yates permutations from the same stream (randomize.py:118-127)."""
    gen = as_generator(rng)
    signs = 1.0 - 2.0 * gen.integers(0, 2, size=(3, n)).astype(np.float64)
    perms = np.stack([gen.permutation(n) for _ in range(3)])
    return RandomizationPlan(signs, perms)


def variant_plan(plan: RandomizationPlan, variant: str) -> RandomizationPlan:
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant: {variant!r}")
    if variant == "full":
        return plan
    ident = identity_plan(plan.n)
    if variant == "sign":
        return RandomizationPlan(plan.signs, ident.perms)
    if variant == "perm":
        return RandomizationPlan(ident.signs, plan.perms)
    return ident


def identity_recursive_plan(n: int, Q: int) -> RecursivePlan:
    return RecursivePlan(tuple(identity_plan(n) for _ in range(Q)))


def draw_recursive_plan(n: int, Q: int, rng) -> RecursivePlan:
    gen = as_generator(rng)
    return RecursivePlan(tuple(draw_plan(n, gen) for _ in range(Q)))


def _rescale_factor(f: BilinearFormula) -> float:
    k = kappa(f)
    if k == 1.0:
        raise ValueError("rescale factor undefined: kappa = 1")
    return 1.0 / (1.0 - k)


def hatted_tensors(f: BilinearFormula, plan: RandomizationPlan, rescaled: bool = True):
    """uh[r,k,l] = u[r,p1(k),p2(l)] s1(k) s2(l); vh with (p2, p3); wh with
    (p1, p3) and, when rescaled, one binary64 multiply by 1/(1-kappa)."""
    if plan.n != f.n:
        raise ValueError("plan and formula grid sizes differ")
    (s1, s2, s3), (p1, p2, p3) = plan.signs, plan.perms
    uh = f.u[:, p1][:, :, p2] * np.outer(s1, s2)[None]
    vh = f.v[:, p2][:, :, p3] * np.outer(s2, s3)[None]
    wh = f.w[:, p1][:, :, p3] * np.outer(s1, s3)[None]
    if rescaled:
        wh = wh * _rescale_factor(f)
    return uh, vh, wh


def plan_levels(f: BilinearFormula, plans, mode):
    """(T, R, n, n) coefficient triple for one recursion level of T plans,
    rounded into the mode (randomize.py:199-209)."""
    m = mode_of(mode)
    plans = list(plans)
    if any(p.n != f.n for p in plans):
        raise ValueError("plan and formula grid sizes differ")
    # batched form of hatted_tensors (same operations: exact sign flips and
    # index gathers, then one binary64 multiply of wh by 1/(1-kappa))
    S = np.stack([p.signs for p in plans])            # (T, 3, n)
    P = np.stack([p.perms for p in plans])            # (T, 3, n)
    c = _rescale_factor(f)

    def hat(t, a, b):
        g = t[:, P[:, a][:, :, None], P[:, b][:, None, :]]  # (R, T, n, n)
        g = np.moveaxis(g, 0, 1)                             # (T, R, n, n)
        return g * (S[:, a][:, :, None] * S[:, b][:, None, :])[:, None]

    uh, vh, wh = hat(f.u, 0, 1), hat(f.v, 1, 2), hat(f.w, 0, 2) * c
    # C-contiguous (T, R, n, n): the gathers leave an (R, T, ...) memory order
    # that a dtype conversion preserves, and device uploads keep strides
    return tuple(np.ascontiguousarray(m.array(t)) for t in (uh, vh, wh))


_plan_level_alias = plan_levels  # reference name: _plan_levels


_KNOWN = None


def _known_formulas():
    """(engine id, formula) for every exact +-1 formula with compiled networks."""
    global _KNOWN
    if _KNOWN is None:
        from ._lib import FORMULA_IDS

        _KNOWN = [
            (FORMULA_IDS["strassen"], strassen_formula()),
            (FORMULA_IDS["laderman"], laderman_formula()),
            (FORMULA_IDS["standard2"], standard_formula(2)),
            (FORMULA_IDS["standard3"], standard_formula(3)),
        ]
    return _KNOWN


def plan_formula_id(f: BilinearFormula):
    """Engine id of an exact +-1 formula with compiled networks, else None.

    Such a formula has kappa == 0 exactly, so its rescale factor is 1 and the
    hatted tables are pure signed permutations of the base coefficients."""
    for fid, g in _known_formulas():
        if g.u.shape == f.u.shape and all(
            np.array_equal(getattr(g, x), getattr(f, x)) for x in "uvw"
        ):
            return fid
    return None


def pack_recursive_plans(rplans, Q: int, n: int) -> np.ndarray:
    """(T, Q, 40) packed device records for a list of RecursivePlans."""
    perms = np.stack([np.stack([p.perms for p in rp.levels]) for rp in rplans])
    signs = np.stack([np.stack([p.signs for p in rp.levels]) for rp in rplans])
    T = len(rplans)
    packed = engine.pack_plans(n, perms.reshape(T * Q, 3, n), signs.reshape(T * Q, 3, n))
    return packed.reshape(T, Q, -1)


def _run(f, rplans, A, B, mode, stats):
    depth = rplans[0].depth
    fid = plan_formula_id(f)
    if fid is not None:
        packed = pack_recursive_plans(rplans, depth, f.n)
        return engine.apply_plans(fid, depth, packed, A[None], B[None], mode, stats)
    levels = [plan_levels(f, [rp.levels[q] for rp in rplans], mode) for q in range(depth)]
    return engine.apply_levels(levels, A[None], B[None], mode, stats)


def plan_count(n: int) -> int:
    """Number of distinct plans (2^n)^3 (n!)^3 (randomize.py:277-279)."""
    import math

    return (2 ** n) ** 3 * math.factorial(n) ** 3


def _all_plans(n: int):
    """Every plan, signs lexicographic with +1 first, permutations in
    itertools order (randomize.py:282-290)."""
    import itertools

    sign_rows = list(itertools.product((1.0, -1.0), repeat=n))
    perm_rows = list(itertools.permutations(range(n)))
    for s1, s2, s3, p1, p2, p3 in itertools.product(
        sign_rows, sign_rows, sign_rows, perm_rows, perm_rows, perm_rows
    ):
        yield RandomizationPlan(np.array([s1, s2, s3]), np.array([p1, p2, p3]))


def all_plan_arrays(n: int):
    """perms (count, 3, n) int64 and signs (count, 3, n) float64 of every plan
    in the enumeration order of _all_plans (randomize.py:282-290:
    itertools.product(signs x3, perms x3), the last factor fastest), built
    with array indexing instead of one RandomizationPlan per plan (110,592
    objects at n = 3)."""
    import itertools

    S = np.array(list(itertools.product((1.0, -1.0), repeat=n)))     # (2^n, n)
    P = np.array(list(itertools.permutations(range(n))), dtype=np.int64)  # (n!, n)
    ns, npm = len(S), len(P)
    idx = np.unravel_index(np.arange(plan_count(n)), (ns, ns, ns, npm, npm, npm))
    signs = np.stack([S[idx[0]], S[idx[1]], S[idx[2]]], axis=1)
    perms = np.stack([P[idx[3]], P[idx[4]], P[idx[5]]], axis=1)
    return perms, signs


def _hatted_batch(f, perms, signs, m):
    """plan_levels over plan arrays (the same gathers and exact sign flips)."""
    c = _rescale_factor(f)

    def hat(t, a, b):
        g = t[:, perms[:, a][:, :, None], perms[:, b][:, None, :]]
        g = np.moveaxis(g, 0, 1)
        return g * (signs[:, a][:, :, None] * signs[:, b][:, None, :])[:, None]

    return tuple(np.ascontiguousarray(m.array(t))
                 for t in (hat(f.u, 0, 1), hat(f.v, 1, 2), hat(f.w, 0, 2) * c))


def enumerate_expectation(f, A, B, mode=DOUBLE, chunk_elements: int = DEFAULT_CHUNK_ELEMENTS,
                          device="cuda:0") -> np.ndarray:
    """Exact expectation of the single-level randomized product over every
    plan (randomize.py:293-334), on the device: plans are evaluated in
    batches and accumulated sequentially in binary64 in enumeration order;
    the average is total / count.  The plan set is built as arrays
    (all_plan_arrays) and packed per batch; ``chunk_elements`` bounds the
    batch the same way as the reference (values never depend on it)."""
    import torch

    from .multiply import _as_operands, _check_blocked

    count = plan_count(f.n)
    if count > 1_000_000:
        raise ValueError(f"{count} plans exceed the enumeration budget")
    m = mode_of(mode)
    A, B = _as_operands(A, B, m)
    _check_blocked(A, B, f.n, 1)
    _rescale_factor(f)
    N = A.shape[0]
    per_trial = max(1, N * N * f.rank // (f.n * f.n))
    chunk = max(1, int(chunk_elements) // per_trial)
    eng = engine.DeviceEngine(m, device=device)
    dev = eng.device
    a = torch.from_numpy(np.ascontiguousarray(A)[None]).to(dev)
    b = torch.from_numpy(np.ascontiguousarray(B)[None]).to(dev)
    total = torch.zeros(N * N, dtype=torch.float64, device=dev)
    fid = plan_formula_id(f)
    tdt = {np.float64: torch.float64, np.float32: torch.float32, np.float16: torch.float16}[m.dtype]
    perms, signs = all_plan_arrays(f.n)
    nf_any = torch.zeros(1, dtype=torch.uint8, device=dev)
    for c0 in range(0, count, chunk):
        P, S = perms[c0:c0 + chunk], signs[c0:c0 + chunk]
        T = len(P)
        out = torch.empty((T, N, N), dtype=tdt, device=dev)
        nf = torch.zeros(T, dtype=torch.uint8, device=dev)
        if fid is not None:
            packed = engine.pack_plans(f.n, P, S).reshape(T, 1, -1)
            eng.apply_plans(fid, 1, torch.from_numpy(packed).to(dev), a, b, out, nf)
        else:
            lv = [tuple(torch.from_numpy(t).to(dev) for t in _hatted_batch(f, P, S, m))]
            eng.apply_levels(lv, a, b, out, nf)
        nf_any |= nf.max().reshape(1)
        eng.sum_trials(out, total)
    torch.cuda.synchronize(dev)
    if bool(nf_any.item()):
        raise OverflowError(f"result left the {m.kind} range")
    return total.cpu().numpy().reshape(N, N) / float(count)


def randomized_apply(f, plan, A, B, mode=DOUBLE, stats=None) -> np.ndarray:
    A, B = _as_operands(A, B, mode)
    _check_blocked(A, B, f.n, 1)
    if plan.n != f.n:
        raise ValueError("plan and formula grid sizes differ")
    _rescale_factor(f)
    return _run(f, [RecursivePlan((plan,))], A, B, mode, stats)[0]


def recursive_randomized_apply(f, rplan, A, B, mode=DOUBLE, stats=None) -> np.ndarray:
    A, B = _as_operands(A, B, mode)
    _check_blocked(A, B, f.n, rplan.depth)
    if rplan.n != f.n:
        raise ValueError("plan and formula grid sizes differ")
    _rescale_factor(f)
    return _run(f, [rplan], A, B, mode, stats)[0]


def recursive_randomized_apply_many(
    f, rplans, A, B, mode=DOUBLE, chunk_elements: int = DEFAULT_CHUNK_ELEMENTS, stats=None
) -> np.ndarray:
    """(len(rplans), s, s) stack; slice t equals recursive_randomized_apply
    with rplans[t] (randomize.py:242-274).  ``chunk_elements`` is accepted
    for API compatibility; the engine chunks trials by device memory, which
    (like the reference's chunking) never changes values."""
    rplans = list(rplans)
    if not rplans:
        raise ValueError("need at least one plan")
    depth = rplans[0].depth
    if any(rp.depth != depth for rp in rplans):
        raise ValueError("plans must share one depth")
    A, B = _as_operands(A, B, mode)
    _check_blocked(A, B, f.n, depth)
    if rplans[0].n != f.n:
        raise ValueError("plan and formula grid sizes differ")
    _rescale_factor(f)
    del chunk_elements
    return _run(f, rplans, A, B, mode, stats)
