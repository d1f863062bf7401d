"""Binary arithmetic modes understood by the B200 engine.

Mirrors the binary part of ``randbc.precision.ScalarMode``
(reference ``pkg/src/randbc/precision.py:50-162``): a mode fixes the storage
dtype and the rounding of every scalar operation (IEEE round-to-nearest-even,
one rounding per multiply and per add).  ``array`` rounds binary64 data into
the mode and raises exactly like the reference (``precision.py:131-152``):
``ValueError`` for non-finite input, ``OverflowError`` when rounding leaves
the mode's range.

``HALF`` is a builder extension: the reference has no binary16
mode, and config 4 of BASELINE.json needs one.  numpy float16 arithmetic is
correctly rounded per operation (float32 intermediates; double rounding is
innocuous because 24 >= 2*11+2), which is what CUDA ``__hmul``/``__hadd``
compute, so the half kind is bit-comparable between the oracle and the GPU.

The decimal toy machine of the reference is out of scope: object
dtype Decimal arithmetic is not a GPU workload.  Passing a decimal mode to the
engine raises ``NotImplementedError``.
"""

from __future__ import annotations

from contextlib import nullcontext
from dataclasses import dataclass

import numpy as np

__all__ = ["Mode", "DOUBLE", "SINGLE", "HALF", "mode_of", "dtype_code", "parse_precision"]

_KINDS = {
    # kind: (numpy dtype, unit roundoff, label, C-ABI dtype code)
    "double": (np.float64, 2.0 ** -53, "f64", 0),
    "single": (np.float32, 2.0 ** -24, "f32", 1),
    "half": (np.float16, 2.0 ** -11, "f16", 2),
}


@dataclass(frozen=True)
class Mode:
    """One binary arithmetic environment (kind in double/single/half)."""

    kind: str

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise ValueError(f"unknown mode kind: {self.kind!r}")

    @property
    def dtype(self):
        return _KINDS[self.kind][0]

    @property
    def epsilon_machine(self) -> float:
        return _KINDS[self.kind][1]

    @property
    def label(self) -> str:
        return _KINDS[self.kind][2]

    @property
    def digits(self):
        return None

    # the reference engine enters these around its ufunc calls; binary modes
    # need no context (precision.py:116-126)
    def context(self):
        return nullcontext()

    def product_context(self):
        return nullcontext()

    def zero(self):
        return 0.0

    def array(self, a) -> np.ndarray:
        """Round array-like data into the mode (idempotent, never aliases)."""
        x = np.asarray(a, dtype=np.float64)
        if not np.all(np.isfinite(x)):
            raise ValueError("input contains non-finite entries")
        if self.kind == "double":
            return x.copy() if x is a else x
        with np.errstate(over="ignore"):
            y = x.astype(self.dtype)
        if not np.all(np.isfinite(y)):
            raise OverflowError(f"value outside {self.label} range")
        return y

    def to_double(self, a) -> np.ndarray:
        return np.asarray(a, dtype=np.float64)


DOUBLE = Mode("double")
SINGLE = Mode("single")
HALF = Mode("half")


def mode_of(mode) -> Mode:
    """Map any duck-typed mode (ours or ``randbc.precision.ScalarMode``) to
    a binary ``Mode``; the decimal kind is rejected as out of scope."""
    kind = getattr(mode, "kind", None)
    if kind == "decimal":
        raise NotImplementedError(
            "decimal (object dtype) arithmetic is not supported by the B200 engine"
        )
    if kind not in _KINDS:
        raise ValueError(f"unsupported arithmetic mode: {mode!r}")
    return Mode(kind)


def dtype_code(mode) -> int:
    return _KINDS[mode_of(mode).kind][3]


def parse_precision(token: str) -> Mode:
    for kind, (_, _, label, _) in _KINDS.items():
        if token == label:
            return Mode(kind)
    raise ValueError(f"bad precision token: {token!r}")
