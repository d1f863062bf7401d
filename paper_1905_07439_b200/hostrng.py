"""Seed derivation and plan draws through the native host RNG (librbc.so,
csrc/hostrng.cu): the reference's ``derive_seed`` / ``derive_rng`` keys
(rng.py:20-29) and ``draw_plan`` (randomize.py:118-127) for many streams at
once, bit-identical to numpy, in microseconds instead of the ~15 us per
stream of Python's SeedSequence.  Used by the device input generator and the
fresh-input trial runs; the host mirror (rng.py, randomize.py) keeps the
numpy objects for everything else."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

__all__ = ["derive_seeds", "philox_keys", "draw_plans"]


def _seeds(seed, count):
    """(array, stride): one seed for all streams (stride 0) or one per stream."""
    if np.ndim(seed) == 0:
        return np.array([int(seed)], dtype=np.uint64), 0
    arr = np.ascontiguousarray([int(s) for s in seed], dtype=np.uint64)
    if len(arr) != count:
        raise ValueError("need one seed per path")
    return arr, 1


def _paths(paths):
    paths = [tuple(int(x) for x in p) for p in paths]
    depth = len(paths[0]) if paths else 0
    if any(len(p) != depth for p in paths):
        raise ValueError("paths must share one depth")
    arr = np.array(paths, dtype=np.uint64).reshape(len(paths), depth)
    return np.ascontiguousarray(arr), depth


def derive_seeds(seed, paths) -> np.ndarray:
    """[derive_seed(seed, *p) for p in paths] as a uint64 array (``seed``: one
    int, or one per path)."""
    arr, depth = _paths(paths)
    sd, ss = _seeds(seed, len(arr))
    out = np.zeros(len(arr), dtype=np.uint64)
    _lib.check(_lib.load().rbc_derive_seeds(sd.ctypes.data, ss, depth, arr.ctypes.data, len(arr),
                                            out.ctypes.data))
    return out


def philox_keys(seed, paths) -> np.ndarray:
    """(len(paths), 2) uint64 Philox keys of derive_rng(seed, *p)."""
    arr, depth = _paths(paths)
    sd, ss = _seeds(seed, len(arr))
    out = np.zeros((len(arr), 2), dtype=np.uint64)
    _lib.check(_lib.load().rbc_philox_keys(sd.ctypes.data, ss, depth, arr.ctypes.data, len(arr),
                                           out.ctypes.data))
    return out


def draw_plans(n: int, seed, paths):
    """perms (count, 3, n) int64 and signs (count, 3, n) float64 of
    draw_plan(n, derive_rng(seed, *p)) for every path."""
    arr, depth = _paths(paths)
    sd, ss = _seeds(seed, len(arr))
    perms = np.zeros((len(arr), 3, n), dtype=np.int64)
    signs = np.zeros((len(arr), 3, n), dtype=np.float64)
    _lib.check(_lib.load().rbc_draw_plans(int(n), sd.ctypes.data, ss, depth, arr.ctypes.data,
                                          len(arr), perms.ctypes.data, signs.ctypes.data))
    return perms, signs
