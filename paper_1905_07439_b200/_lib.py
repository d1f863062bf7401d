"""ctypes binding of librbc.so (C ABI declared in include/rbc.h).

The library is loaded lazily on first use.  There is no CPU fallback: if the
shared library is missing or no CUDA device is present, calls raise
``RuntimeError`` instead of computing anything elsewhere.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "librbc.so"

RBC_OK = 0
RBC_EVALUE = 1
RBC_EOVERFLOW = 2
RBC_ERUNTIME = 3
RBC_EUNSUPPORTED = 4

PLAN_BYTES = 40

FORMULA_IDS = {"strassen": 1, "laderman": 2, "standard2": 3, "standard3": 4}

# Every symbol include/rbc.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = (
    "rbc_abi_version",
    "rbc_last_error",
    "rbc_device_count",
    "rbc_release_device_memory",
    "rbc_profile_enable",
    "rbc_profile_summary",
    "rbc_apply_levels",
    "rbc_leaf_matmul",
    "rbc_pack_plans",
    "rbc_apply_plans",
    "rbc_levels_workspace_bytes",
    "rbc_apply_levels_async",
    "rbc_plans_workspace_bytes",
    "rbc_apply_plans_async",
    "rbc_leaf_matmul_async",
    "rbc_truth_async",
    "rbc_rel_errors_scratch_bytes",
    "rbc_rel_errors_async",
    "rbc_rel_errors",
    "rbc_nonfinite_async",
    "rbc_error_trials",
    "rbc_error_trials_begin",
    "rbc_error_trials_end",
    "rbc_error_trials_workspace_bytes",
    "rbc_error_trials_async",
    "rbc_average_trials_workspace_bytes",
    "rbc_average_trials_async",
    "rbc_sum_trials_async",
    "rbc_matgen",
    "rbc_rescaled_multiply",
    "rbc_derive_seeds",
    "rbc_philox_keys",
    "rbc_draw_plans",
)

_lock = threading.Lock()
_lib = None

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_size = ctypes.c_size_t
c_vp = ctypes.c_void_p
c_u64p = ctypes.POINTER(ctypes.c_uint64)


def _declare(lib):
    P = ctypes.POINTER
    sig = {
        "rbc_abi_version": (c_int, []),
        "rbc_last_error": (ctypes.c_char_p, []),
        "rbc_device_count": (c_int, []),
        "rbc_release_device_memory": (c_int, []),
        "rbc_profile_enable": (None, [c_int]),
        "rbc_profile_summary": (c_i64, [ctypes.c_char_p, c_size]),
        "rbc_apply_levels": (
            c_int,
            [c_int, c_int, P(c_i32), P(c_i32), P(c_i64), P(c_vp), P(c_vp), P(c_vp),
             c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_u64p],
        ),
        "rbc_leaf_matmul": (c_int, [c_int, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
        "rbc_rel_errors": (c_int, [c_int, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp]),
        "rbc_pack_plans": (c_int, [c_int, c_i64, c_vp, c_vp, c_vp]),
        "rbc_apply_plans": (
            c_int,
            [c_int, c_int, c_int, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_u64p],
        ),
        "rbc_levels_workspace_bytes": (c_size, [c_int, c_int, P(c_i32), P(c_i32), c_i64, c_i64]),
        "rbc_apply_levels_async": (
            c_int,
            [c_int, c_int, P(c_i32), P(c_i32), P(c_i64), P(c_vp), P(c_vp), P(c_vp),
             c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_size, c_vp],
        ),
        "rbc_plans_workspace_bytes": (c_size, [c_int, c_int, c_int, c_i64, c_i64]),
        "rbc_apply_plans_async": (
            c_int,
            [c_int, c_int, c_int, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp,
             c_vp, c_size, c_vp],
        ),
        "rbc_leaf_matmul_async": (
            c_int, [c_int, c_int, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]
        ),
        "rbc_truth_async": (c_int, [c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
        "rbc_rel_errors_scratch_bytes": (c_size, [c_i64]),
        "rbc_rel_errors_async": (c_int, [c_int, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
        "rbc_nonfinite_async": (c_int, [c_int, c_i64, c_i64, c_vp, c_vp, c_vp]),
        "rbc_sum_trials_async": (c_int, [c_int, c_i64, c_i64, c_vp, c_vp, c_vp]),
        "rbc_matgen": (c_int, [c_int, c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
        "rbc_error_trials": (
            c_int,
            [c_int, c_int, c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp],
        ),
        "rbc_error_trials_begin": (
            c_int,
            [c_int, c_int, c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp,
             P(c_i64)],
        ),
        "rbc_error_trials_end": (c_int, [c_i64]),
        "rbc_error_trials_workspace_bytes": (c_size, [c_int, c_int, c_int, c_i64, c_i64]),
        "rbc_average_trials_workspace_bytes": (c_size, [c_int, c_int, P(c_i32), P(c_i32), c_i64, c_i64]),
        "rbc_average_trials_async": (
            c_int,
            [c_int, c_int, P(c_i32), P(c_i32), c_i64, c_i64, c_i64, c_vp, c_vp,
             P(c_vp), P(c_vp), P(c_vp), P(c_vp), P(c_vp), P(c_vp), c_int, P(c_i32),
             c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp],
        ),
        "rbc_derive_seeds": (c_int, [c_vp, c_i64, c_int, c_vp, c_i64, c_vp]),
        "rbc_philox_keys": (c_int, [c_vp, c_i64, c_int, c_vp, c_i64, c_vp]),
        "rbc_draw_plans": (c_int, [c_int, c_vp, c_i64, c_int, c_vp, c_i64, c_vp, c_vp]),
        "rbc_rescaled_multiply": (
            c_int,
            [c_int, c_int, c_int, P(c_i32), P(c_i32), P(c_vp), P(c_vp), P(c_vp), c_int, P(c_i32),
             c_i64, c_vp, c_vp, c_vp],
        ),
        "rbc_error_trials_async": (
            c_int,
            [c_int, c_int, c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
             c_vp, c_size, c_vp],
        ),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def load(path: os.PathLike | None = None):
    """Load (once) and return the ctypes handle of librbc.so."""
    global _lib
    with _lock:
        if _lib is None:
            p = Path(path) if path else LIB_PATH
            if not p.exists():
                raise RuntimeError(
                    f"{p} is missing: build it with `python -m paper_1905_07439_b200.build` "
                    "(the engine has no CPU fallback)"
                )
            _lib = _declare(ctypes.CDLL(str(p)))
        return _lib


def last_error() -> str:
    msg = load().rbc_last_error()
    return msg.decode() if msg else ""


def check(rc: int, *, overflow_msg: str | None = None) -> None:
    """Map a C ABI status to the reference's exception types."""
    if rc == RBC_OK:
        return
    msg = last_error()
    if rc == RBC_EVALUE:
        raise ValueError(msg)
    if rc == RBC_EOVERFLOW:
        raise OverflowError(overflow_msg or msg)
    if rc == RBC_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg or f"librbc status {rc}")


def profile_enable(on: bool = True) -> None:
    load().rbc_profile_enable(1 if on else 0)


def profile_summary() -> dict:
    """{stage: {count, ms, bytes, flops}} of the launches since profile_enable."""
    import json

    lib = load()
    need = lib.rbc_profile_summary(None, 0)
    buf = ctypes.create_string_buffer(int(need) + 16)
    lib.rbc_profile_summary(buf, len(buf))
    return json.loads(buf.value.decode())


def require_device() -> None:
    if load().rbc_device_count() < 1:
        raise RuntimeError("librbc: no CUDA device visible (the engine has no CPU fallback)")
