"""Bilinear formulas (U, V, W) as dense (R, n, n) binary64 tensors.

Host-side mirror of ``randbc.formula`` (reference ``pkg/src/randbc/formula.py``):

* ``BilinearFormula``        -- formula.py:45-82 (frozen, read-only tensors)
* ``strassen_formula``       -- formula.py:98-114 (same 7 terms, same order)
* ``standard_formula``       -- formula.py:117-137
* ``perturb``                -- formula.py:140-173 (same draw order)
* ``kappa``                  -- formula.py:176-194 (sequential binary64 loops)
* ``is_exact``               -- formula.py:222-227
* ``format_formula`` / ``parse_formula`` -- the ``bilinear-formula v1`` text
  format of formula.py:249-313

Builder extensions the BASELINE configs need:

* ``laderman_formula``       -- Laderman's exact <3,3,3;23> formula (1976),
  cited by the paper at PAPER.md:27; shipped as ``formulas/laderman.txt`` and
  gated by ``is_exact`` and ``kappa == 0``.
* ``perturb_all``            -- N(0, sigma) noise on *every* coefficient, drawn
  as one ``normal(0, sigma, (3, R, n, n))`` block in u, v, w order (config 3).
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .rng import as_generator

__all__ = [
    "BilinearFormula",
    "strassen_formula",
    "standard_formula",
    "laderman_formula",
    "perturb",
    "perturb_all",
    "kappa",
    "is_exact",
    "format_formula",
    "parse_formula",
    "load_formula",
    "save_formula",
]

_FORMULA_DIR = Path(__file__).resolve().parent / "formulas"


@dataclass(frozen=True)
class BilinearFormula:
    """C_ij = sum_r w[r,i,j] (sum_kl u[r,k,l] A_kl)(sum_kl v[r,k,l] B_kl)."""

    u: np.ndarray
    v: np.ndarray
    w: np.ndarray

    def __post_init__(self):
        frozen = {}
        for name in ("u", "v", "w"):
            t = np.array(getattr(self, name), dtype=np.float64)
            if t.ndim != 3:
                raise ValueError(f"{name} must have shape (R, n, n)")
            if not np.all(np.isfinite(t)):
                raise ValueError(f"{name} contains non-finite coefficients")
            t.flags.writeable = False
            frozen[name] = t
        if not frozen["u"].shape == frozen["v"].shape == frozen["w"].shape:
            raise ValueError("u, v, w must share one shape")
        R, n, n2 = frozen["u"].shape
        if n != n2:
            raise ValueError("block grid must be square")
        if R < 1 or n < 1:
            raise ValueError("need at least one term and one block")
        for name, t in frozen.items():
            object.__setattr__(self, name, t)

    @property
    def n(self) -> int:
        return self.u.shape[1]

    @property
    def rank(self) -> int:
        return self.u.shape[0]


def _from_terms(n: int, terms) -> BilinearFormula:
    """Build a formula from per-term {(row, col): coeff} maps (0-based)."""
    R = len(terms)
    out = np.zeros((3, R, n, n))
    for r, triple in enumerate(terms):
        for which, entries in enumerate(triple):
            for (k, l), c in entries.items():
                out[which, r, k, l] = c
    return BilinearFormula(out[0], out[1], out[2])


def _grid(rows):
    return {(k, l): c for k, row in enumerate(rows) for l, c in enumerate(row) if c}


# Strassen's 7 products in the reference's term order (formula.py:98-106);
# each entry is the (u, v, w) 2x2 coefficient grid of one term.
_STRASSEN = (
    ([[1, 0], [0, 1]], [[1, 0], [0, 1]], [[1, 0], [0, 1]]),
    ([[0, 0], [1, 1]], [[1, 0], [0, 0]], [[0, 0], [1, -1]]),
    ([[1, 0], [0, 0]], [[0, 1], [0, -1]], [[0, 1], [0, 1]]),
    ([[0, 0], [0, 1]], [[-1, 0], [1, 0]], [[1, 0], [1, 0]]),
    ([[1, 1], [0, 0]], [[0, 0], [0, 1]], [[-1, 1], [0, 0]]),
    ([[-1, 0], [1, 0]], [[1, 1], [0, 0]], [[0, 0], [0, 1]]),
    ([[0, 1], [0, -1]], [[0, 0], [1, 1]], [[1, 0], [0, 0]]),
)


def strassen_formula() -> BilinearFormula:
    return _from_terms(2, [tuple(_grid(g) for g in t) for t in _STRASSEN])


def standard_formula(n: int) -> BilinearFormula:
    """n^3 inner-product terms, term (i, l, j) with i slowest (formula.py:117-137)."""
    if n < 1:
        raise ValueError("n must be positive")
    terms = []
    for i in range(n):
        for l in range(n):
            for j in range(n):
                terms.append(({(i, l): 1.0}, {(l, j): 1.0}, {(i, j): 1.0}))
    return _from_terms(n, terms)


def laderman_formula() -> BilinearFormula:
    """Laderman's exact 23-term 3x3 formula, loaded from formulas/laderman.txt."""
    f = load_formula(_FORMULA_DIR / "laderman.txt")
    if f.n != 3 or f.rank != 23 or not is_exact(f) or kappa(f) != 0.0:
        raise RuntimeError("formulas/laderman.txt is not an exact <3,3,3;23> formula")
    return f


def perturb(f: BilinearFormula, sigma: float, extra_zeros: int, rng) -> BilinearFormula:
    """Reference perturbation (formula.py:140-173): per tensor u, v, w in turn,
    N(0, sigma) noise on every coefficient equal to 1, then on ``extra_zeros``
    distinct zero coefficients chosen uniformly (draw order: ones-noise,
    zero-position choice, zeros-noise)."""
    if sigma <= 0.0:
        raise ValueError("sigma must be positive")
    if extra_zeros < 0:
        raise ValueError("extra_zeros must be >= 0")
    gen = as_generator(rng)
    tensors = (f.u, f.v, f.w)
    for name, t in zip("uvw", tensors):
        if extra_zeros > int(np.count_nonzero(t == 0.0)):
            raise ValueError(f"tensor {name} has fewer than {extra_zeros} zero entries")
    noisy = []
    for t in tensors:
        flat = t.ravel().copy()
        at_one = np.flatnonzero(flat == 1.0)
        flat[at_one] += gen.normal(0.0, sigma, size=at_one.size)
        at_zero = np.flatnonzero(flat == 0.0)
        if extra_zeros:
            chosen = at_zero[gen.choice(at_zero.size, size=extra_zeros, replace=False)]
            flat[chosen] += gen.normal(0.0, sigma, size=extra_zeros)
        noisy.append(flat.reshape(t.shape))
    return BilinearFormula(*noisy)


def perturb_all(f: BilinearFormula, sigma: float, rng) -> BilinearFormula:
    """Builder extension for config 3: i.i.d. N(0, sigma) on every entry of
    u, v and w, drawn as ``normal(0, sigma, (3, R, n, n))`` in u, v, w order."""
    if sigma <= 0.0:
        raise ValueError("sigma must be positive")
    gen = as_generator(rng)
    noise = gen.normal(0.0, sigma, size=(3,) + f.u.shape)
    return BilinearFormula(f.u + noise[0], f.v + noise[1], f.w + noise[2])


_KAPPA_CACHE: dict = {}


def kappa(f: BilinearFormula) -> float:
    """n^-3 * sum_(i,j,l) (1 - sum_r u[r,i,l] v[r,l,j] w[r,i,j]), accumulated
    sequentially in binary64, (i, j, l) lexicographic, r innermost
    (formula.py:176-194).  The order is part of the contract: the rescale
    factor 1/(1-kappa) must round exactly as the reference's does.

    Formulas are immutable, so the value is memoised by coefficient bytes
    (the reference recomputes it for every hatted table)."""
    key = (f.u.shape, f.u.tobytes(), f.v.tobytes(), f.w.tobytes())
    hit = _KAPPA_CACHE.get(key)
    if hit is not None:
        return hit
    val = _kappa_sequential(f)
    if len(_KAPPA_CACHE) > 256:
        _KAPPA_CACHE.clear()
    _KAPPA_CACHE[key] = val
    return val


def _kappa_sequential(f: BilinearFormula) -> float:
    u = f.u.tolist()
    v = f.v.tolist()
    w = f.w.tolist()
    n, R = f.n, f.rank
    total = 0.0
    for i in range(n):
        for j in range(n):
            for l in range(n):
                s = 0.0
                for r in range(R):
                    s += u[r][i][l] * v[r][l][j] * w[r][i][j]
                total += 1.0 - s
    return float(total) / float(n ** 3)


def is_exact(f: BilinearFormula, tol: float = 0.0) -> bool:
    """Brent equations hold within tol (formula.py:222-227)."""
    if tol < 0.0:
        raise ValueError("tol must be >= 0")
    n = f.n
    got = np.einsum("rkl,rmp,rij->klmpij", f.u, f.v, f.w, optimize=True)
    d = np.eye(n)
    want = np.einsum("ki,pj,lm->klmpij", d, d, d)
    return bool(np.max(np.abs(got - want)) <= tol)


_MAGIC = "bilinear-formula v1"


def format_formula(f: BilinearFormula) -> str:
    out = [_MAGIC, f"n {f.n}", f"R {f.rank}"]
    for name in "uvw":
        out.append(f"tensor {name}")
        t = getattr(f, name)
        for r in range(f.rank):
            for row in t[r]:
                out.append(" ".join(repr(float(x)) for x in row))
    return "\n".join(out) + "\n"


def parse_formula(text: str) -> BilinearFormula:
    lines = [ln.strip() for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0] != _MAGIC:
        raise ValueError("not a bilinear-formula v1 document")
    try:
        n = int(lines[1].split()[1])
        R = int(lines[2].split()[1])
    except (IndexError, ValueError):
        raise ValueError("malformed header") from None
    at = 3
    tensors = []
    for name in "uvw":
        if at >= len(lines) or lines[at] != f"tensor {name}":
            raise ValueError(f"expected 'tensor {name}' section")
        at += 1
        if at + R * n > len(lines):
            raise ValueError("truncated tensor section")
        rows = [[float(tok) for tok in lines[at + i].split()] for i in range(R * n)]
        if any(len(row) != n for row in rows):
            raise ValueError(f"expected {n} entries per row")
        tensors.append(np.array(rows).reshape(R, n, n))
        at += R * n
    if at != len(lines):
        raise ValueError("trailing content after tensors")
    return BilinearFormula(*tensors)


def load_formula(path) -> BilinearFormula:
    return parse_formula(Path(path).read_text(encoding="ascii"))


def save_formula(f: BilinearFormula, path) -> None:
    Path(path).write_text(format_formula(f), encoding="ascii")
