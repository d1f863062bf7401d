"""CPU oracle of the diagonal rescaling baseline -- test infrastructure only.

Restates reference ``pkg/src/randbc/rescale.py:36-99`` (``rescaled_multiply``
with the "2x O-I" schedule) element by element, written independently of the
product's host code: every maximum, reciprocal, ratio, square root and
scaled entry is formed one numpy scalar at a time in the mode's dtype, so
each operation rounds exactly once in that dtype (binary16 scalars round via
binary32, which is innocuous for these operations: 24 >= 2*11 + 2).  The
recursion in between is ``oracle.engine.apply_levels`` (the deterministic
formula tables, ``multiply.py:34-41,72-99``).  Only ``tests/`` use it.
"""

from __future__ import annotations

import numpy as np

from . import engine


def _maxabs(vec):
    best = vec.dtype.type(0)
    for x in vec:
        ax = -x if x < 0 else x
        if ax > best:
            best = ax
    return best


def _check(vals, what):
    for v in vals:
        if float(v) == 0.0:
            raise ValueError(f"degenerate input: zero {what} maximum")


def _scaled(X, row=None, col=None):
    """New array: X[i, j] * row[i] (one rounding), then * col[j]."""
    out = X.copy()
    n = X.shape[0]
    for i in range(n):
        for j in range(n):
            v = out[i, j]
            if row is not None:
                v = row[i] * v
            if col is not None:
                v = v * col[j]
            out[i, j] = v
    return out


def rescaled_multiply(A, B, Q, schedule, mode, u, v, w):
    """A, B: mode-typed (N, N); (u, v, w): the formula's (R, n, n) tables in
    the mode.  Returns the mode-typed product; raises like the reference."""
    dt = np.dtype(mode.dtype).type
    A = np.array(A, dtype=dt)
    B = np.array(B, dtype=dt)
    n = A.shape[0]
    one = dt(1)
    undo = []
    for step in schedule:
        if step == "outside":
            ra = [_maxabs(A[i, :]) for i in range(n)]
            _check(ra, "row")
            cb = [_maxabs(B[:, j]) for j in range(n)]
            _check(cb, "column")
            A = _scaled(A, row=[dt(one / x) for x in ra])
            B = _scaled(B, col=[dt(one / x) for x in cb])
            undo.append((ra, cb))
        elif step == "inside":
            rb = [_maxabs(B[i, :]) for i in range(n)]
            _check(rb, "row")
            ca = [_maxabs(A[:, j]) for j in range(n)]
            _check(ca, "column")
            d = [dt(np.sqrt(dt(rb[k] / ca[k]))) for k in range(n)]
            A = _scaled(A, col=d)
            B = _scaled(B, row=[dt(one / x) for x in d])
        else:
            raise ValueError(f"unknown schedule step: {step!r}")
    with np.errstate(all="ignore"):
        if Q == 0:
            C = engine.standard_multiply(A, B)
        else:
            C = engine.apply_levels([(u[None], v[None], w[None])] * Q, A[None], B[None], mode)[0]
        for ra, cb in reversed(undo):
            C = _scaled(C, row=ra, col=cb)
    return C
