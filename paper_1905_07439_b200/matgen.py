"""Seeded test-matrix pairs (host side, binary64).

Mirror of ``randbc.matgen.generate`` (reference ``pkg/src/randbc/matgen.py:55-97``):
A is drawn from ``derive_rng(seed, 0)`` and B from ``derive_rng(seed, 1)``.

Reference kinds: gaussian, uniform, adv1, adv2, adv3, hilbert.
Builder kinds for the BASELINE configs, drawn on the same
streams:

* ``uniform_pm1``   -- ``2 * random() - 1`` entries (config 2)
* ``quadrant100``   -- standard normal, then A[:N/2, :N/2] *= 100 and
                       B[N/2:, N/2:] *= 100 in binary64 (config 4)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .rng import derive_rng

__all__ = ["MATRIX_KINDS", "BUILDER_KINDS", "MatrixSpec", "generate", "kind_index",
           "philox_key", "generate_device"]

MATRIX_KINDS = ("gaussian", "uniform", "adv1", "adv2", "adv3", "hilbert")
BUILDER_KINDS = ("uniform_pm1", "quadrant100")


def kind_index(kind: str) -> int:
    """Index used in the matrix seed path (experiments.py:237-239); builder
    kinds reuse the index of the reference family they derive from."""
    base = {"uniform_pm1": "uniform", "quadrant100": "gaussian"}.get(kind, kind)
    return MATRIX_KINDS.index(base)


@dataclass(frozen=True)
class MatrixSpec:
    kind: str
    size: int
    seed: int = 0

    def __post_init__(self):
        if self.kind not in MATRIX_KINDS + BUILDER_KINDS:
            raise ValueError(f"unknown matrix kind: {self.kind!r}")
        if self.size < 1:
            raise ValueError("size must be >= 1")
        if self.kind.startswith("adv") and self.size < 2:
            raise ValueError("adversarial kinds need size >= 2")
        if not 0 <= int(self.seed) < 2 ** 64:
            raise ValueError("seed must fit in u64")


def generate(spec: MatrixSpec):
    n = spec.size
    ga = derive_rng(spec.seed, 0)
    gb = derive_rng(spec.seed, 1)
    kind = spec.kind
    if kind in ("gaussian", "quadrant100"):
        A, B = ga.standard_normal((n, n)), gb.standard_normal((n, n))
        if kind == "quadrant100":
            h = n // 2
            A[:h, :h] *= 100.0
            B[h:, h:] *= 100.0
        return A, B
    if kind == "uniform":
        return ga.random((n, n)), gb.random((n, n))
    if kind == "uniform_pm1":
        return 2.0 * ga.random((n, n)) - 1.0, 2.0 * gb.random((n, n)) - 1.0
    i = np.arange(1, n + 1, dtype=np.float64)[:, None]
    j = np.arange(1, n + 1, dtype=np.float64)[None, :]
    if kind == "hilbert":
        H = 1.0 / (i + j - 1.0)
        return H, H.copy()
    half = n / 2.0
    tiny = 1.0 / (n * n)
    huge = float(n * n)
    ones = np.ones((n, n))
    if kind == "adv1":
        sa = np.where(j > half, tiny, 1.0) * ones
        sb = np.where(i < half, tiny, 1.0) * ones
    elif kind == "adv2":
        sa = np.where((i < half) & (j > half), huge, 1.0) * ones
        sb = np.where(j < half, tiny, 1.0) * ones
    else:
        band = ((i < half) & (j > half)) | ((i >= half) & (j <= half))
        sa = np.where(band, tiny, 1.0) * ones
        sb = sa
    return ga.random(sa.shape) * sa, gb.random(sb.shape) * sb


def philox_key(seed: int, *path: int) -> tuple[int, int]:
    """The 128-bit Philox key of ``derive_rng(seed, *path)`` (reference
    rng.py:20-23): numpy's SeedSequence hashing, evaluated on the host."""
    ss = np.random.SeedSequence(int(seed), spawn_key=tuple(int(p) for p in path))
    key = np.random.Philox(ss).state["state"]["key"]
    return int(key[0]), int(key[1])


def generate_device(kind: str, size: int, seeds, mode, device="cuda:0", which=(0, 1), out=None):
    """Device twin of :func:`generate` over many seeds: returns a tuple of
    torch tensors, one per entry of ``which`` (0 = A, 1 = B), each
    (len(seeds), size, size) in the mode dtype on ``device``, bit-identical to
    ``mode.array(generate(MatrixSpec(kind, size, seed))[w])`` (librbc
    rbc_matgen: Philox4x64-10 and numpy's ziggurat on the device, SURVEY §8f
    rank 4).  Raises OverflowError where the rounding into the mode overflows,
    like ``mode.array``.  ``out``: optional tensors (one per ``which``) to
    draw into instead of allocating."""
    import ctypes

    import torch

    from . import _lib, hostrng
    from .precision import dtype_code, mode_of

    if kind not in MATRIX_KINDS + BUILDER_KINDS:
        raise ValueError(f"unknown matrix kind: {kind!r}")
    m = mode_of(mode)
    seeds = [int(s) for s in seeds]
    for sd in seeds:
        MatrixSpec(kind, size, sd)  # same validation as the host path
    tdt = {"double": torch.float64, "single": torch.float32, "half": torch.float16}[m.kind]
    dev = torch.device(device)
    lib = _lib.load()
    code = (MATRIX_KINDS + BUILDER_KINDS).index(kind)
    outs = []
    dst = list(out) if out is not None else [None] * len(which)
    for w, buf in zip(which, dst):
        shape = (len(seeds), size, size)
        if buf is not None and (tuple(buf.shape) != shape or buf.dtype != tdt or not buf.is_contiguous()):
            raise ValueError("out tensor does not match the draw")
        out = buf if buf is not None else torch.empty(shape, dtype=tdt, device=dev)
        flags = torch.zeros(max(1, len(seeds)), dtype=torch.uint8, device=dev)
        for c0 in range(0, len(seeds), 65535):
            part = seeds[c0:c0 + 65535]
            keys = hostrng.philox_keys(part, [(w,)] * len(part)).reshape(-1)
            wh = np.full(len(part), w, dtype=np.int32)
            with torch.cuda.device(dev):
                st = torch.cuda.current_stream(dev).cuda_stream
                rc = lib.rbc_matgen(code, dtype_code(m), len(part), size,
                                    keys.ctypes.data_as(ctypes.c_void_p),
                                    wh.ctypes.data_as(ctypes.c_void_p),
                                    ctypes.c_void_p(out[c0:].data_ptr()),
                                    ctypes.c_void_p(flags[c0:].data_ptr()), ctypes.c_void_p(st))
            _lib.check(rc)
        if len(seeds) and bool(flags.any()):
            raise OverflowError(f"value outside {m.label} range")
        outs.append(out)
    return tuple(outs)
