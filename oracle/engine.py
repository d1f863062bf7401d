"""CPU oracle for the BC-multiply hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module, and only as the checker or the
timed CPU baseline.  The product path (``paper_1905_07439_b200``) never calls
it; it fails loudly when its CUDA library is missing.

This is a numpy restatement of the reference engine
``randbc._engine`` (``pkg/src/randbc/_engine.py``), written independently but
following the same per-element rounding sequence, so its outputs are
bitwise equal to the reference's:

* ``combine``     <- ``_expand``      (_engine.py:64-90): per output element,
  a left fold over the block column l inside each block row k, then a left
  fold of the row sums over k; every term is one rounded multiply.
* ``leaf``        <- ``leaf_matmul``  (_engine.py:42-61): sequential over the
  shared index, first term initialises, multiply and add rounded separately.
* ``accumulate``  <- ``_contract``    (_engine.py:93-114): left fold over the
  term index r, first term initialises.
* ``apply_levels``<- ``apply_levels`` (_engine.py:117-149), including its
  ValueError / OverflowError behaviour and the ``leaf_multiplies`` counter.

Zero coefficients are multiplied and added like any other term, exactly as in
the reference.  numpy's same-dtype ufuncs round once per operation in
binary64 / binary32, and binary16 is computed through float32 and rounded
once more, which is innocuous (24 >= 2*11 + 2), so all three kinds match an
elementwise IEEE evaluation.

Parity pin: ``tests/test_oracle_golden.py`` checks this module bit-for-bit
against fixtures produced by the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/engine_cases.npz``).
"""

from __future__ import annotations

import numpy as np

__all__ = ["combine", "leaf", "accumulate", "apply_levels", "rel_errors", "standard_multiply"]


def _dtype_of(mode):
    return np.dtype(mode.dtype)


def combine(x: np.ndarray, coeff: np.ndarray) -> np.ndarray:
    """(T0, K, s, s) x (Tc, R, n, n) -> (T, K*R, s/n, s/n), branch = K*R + r."""
    T0, K, s, _ = x.shape
    Tc, R, n, _ = coeff.shape
    mb = s // n
    T = max(T0, Tc)
    # grid view: [t, K, block row k, i, block col l, j]
    grid = x.reshape(T0, K, n, mb, n, mb)
    total = None
    for k in range(n):
        rowsum = None
        for l in range(n):
            c = coeff[:, None, :, k, l, None, None]          # (Tc, 1, R, 1, 1)
            blk = grid[:, :, None, k, :, l, :]                # (T0, K, 1, mb, mb)
            term = np.multiply(c, blk)
            rowsum = term if rowsum is None else np.add(rowsum, term)
        total = rowsum if total is None else np.add(total, rowsum)
    return np.ascontiguousarray(total).reshape(T, K * R, mb, mb)


def leaf(x: np.ndarray, y: np.ndarray, dtype=None) -> np.ndarray:
    """Batched x @ y over the last two axes, k ascending, no fused multiply-add."""
    kdim = x.shape[-1]
    if y.shape[-2] != kdim:
        raise ValueError("inner dimensions do not conform")
    lead = np.broadcast_shapes(x.shape[:-2], y.shape[:-2])
    shape = lead + (x.shape[-2], y.shape[-1])
    if kdim == 0:
        return np.zeros(shape, dtype=dtype if dtype is not None else x.dtype)
    acc = np.broadcast_to(np.multiply(x[..., :, 0:1], y[..., 0:1, :]), shape).copy()
    for k in range(1, kdim):
        np.add(acc, np.multiply(x[..., :, k : k + 1], y[..., k : k + 1, :]), out=acc)
    return acc


def accumulate(children: np.ndarray, coeff: np.ndarray) -> np.ndarray:
    """(T, K, R, mb, mb) x (Tc, R, n, n) -> (T, K, n*mb, n*mb)."""
    T, K, R, mb, _ = children.shape
    n = coeff.shape[-1]
    out = np.empty((T, K, n, mb, n, mb), dtype=children.dtype)
    for i in range(n):
        for j in range(n):
            acc = None
            for r in range(R):
                term = np.multiply(coeff[:, r, i, j][:, None, None, None], children[:, :, r])
                acc = term if acc is None else np.add(acc, term)
            out[:, :, i, :, j, :] = acc
    return out.reshape(T, K, n * mb, n * mb)


def apply_levels(levels, a: np.ndarray, b: np.ndarray, mode, stats=None) -> np.ndarray:
    """Breadth-first evaluation of a Q-level blocked formula recursion."""
    if not levels:
        raise ValueError("need at least one level")
    x = a[:, None]
    y = b[:, None]
    for u, v, _ in levels:
        n = u.shape[-1]
        if x.shape[-1] % n:
            raise ValueError("operand size not divisible by block grid")
        x = combine(x, u)
        y = combine(y, v)
    prod = leaf(x, y)
    if stats is not None:
        stats["leaf_multiplies"] = stats.get("leaf_multiplies", 0) + prod.shape[0] * prod.shape[1]
    for _, _, w in reversed(levels):
        R = w.shape[1]
        T, KR, mb, _ = prod.shape
        prod = accumulate(prod.reshape(T, KR // R, R, mb, mb), w)
    out = prod[:, 0]
    if not np.all(np.isfinite(out)):
        raise OverflowError(f"result left the {mode.kind} range")
    return out


def standard_multiply(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Inner-product algorithm on 2-D operands (reference multiply.py:44-51)."""
    return leaf(A[None], B[None])[0]


def rel_errors(results: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """Per-trial ||C_t - ref||_F / ||ref||_F in binary64
    (reference experiments.py:222-223, 258-261)."""
    res = np.asarray(results, dtype=np.float64)
    diff = res - ref[None]
    refnorm = float(np.linalg.norm(np.asarray(ref, dtype=np.float64).ravel()))
    return np.sqrt(np.sum(diff * diff, axis=(1, 2))) / refnorm
