"""Error trials on the device: binary64 truth, BC products, relative errors.

The per-pair work of the reference's distribution experiments
(experiments.py:248-261, 327-379) as one native call:

* ``error_trials``        -- host buffers in, per-trial errors out
                             (C ABI ``rbc_error_trials``; the public,
                             reference-facing path the e2e number is taken on)
* ``DeviceErrorTrials``   -- the same pipeline on device-resident torch
                             tensors and a caller stream
                             (``rbc_error_trials_async``), for throughput runs
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib, engine
from .precision import dtype_code, mode_of
from .randomize import pack_recursive_plans, plan_formula_id

__all__ = ["error_trials", "identity_packed", "DeviceErrorTrials"]


def identity_packed(n: int, Q: int) -> np.ndarray:
    perms = np.tile(np.arange(n), (Q, 3, 1))
    return engine.pack_plans(n, perms, np.ones((Q, 3, n))).reshape(1, Q, -1)


def _vp(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def error_trials(f, Q: int, A, B, mode, rplans=None, packed=None, with_det: bool = True):
    """Per-trial relative errors of randomized (and deterministic) products.

    A, B   : (T, N, N) operands in the mode (one pair per trial)
    rplans : T RecursivePlans (or ``packed`` (T, Q, 40) records), optional
    returns dict with err_rand, err_det (float64 (T,)), nf_rand, nf_det (bool)
    """
    m = mode_of(mode)
    fid = plan_formula_id(f)
    if fid is None:
        raise NotImplementedError("error_trials supports the exact +-1 formulas (plan path)")
    A = np.ascontiguousarray(A, dtype=m.dtype)
    B = np.ascontiguousarray(B, dtype=m.dtype)
    T, N, _ = A.shape
    if packed is None and rplans is not None:
        packed = pack_recursive_plans(list(rplans), Q, f.n)
    if packed is not None:
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        if packed.shape != (T, Q, _lib.PLAN_BYTES):
            raise ValueError("packed plans must be (T, Q, 40)")
    err_r = np.full(T, np.nan)
    err_d = np.full(T, np.nan)
    nf_r = np.zeros(T, np.uint8)
    nf_d = np.zeros(T, np.uint8)
    rc = _lib.load().rbc_error_trials(
        dtype_code(m), fid, Q, T, N, _vp(A), _vp(B),
        _vp(packed) if packed is not None else None, int(with_det),
        _vp(err_r), _vp(err_d), _vp(nf_r), _vp(nf_d),
    )
    _lib.check(rc)
    out = {}
    if packed is not None:
        out["err_rand"], out["nf_rand"] = err_r, nf_r.astype(bool)
    if with_det:
        out["err_det"], out["nf_det"] = err_d, nf_d.astype(bool)
    return out


class DeviceErrorTrials:
    """Device-resident pipeline over torch CUDA tensors (throughput path)."""

    def __init__(self, f, Q: int, N: int, mode, T: int, device="cuda:0", workspace_bytes=None):
        import torch

        self.torch = torch
        self.m = mode_of(mode)
        self.fid = plan_formula_id(f)
        if self.fid is None:
            raise NotImplementedError("DeviceErrorTrials supports the exact +-1 formulas")
        self.Q, self.N, self.T, self.n = Q, N, T, f.n
        self.device = torch.device(device)
        lib = _lib.load()
        need = lib.rbc_error_trials_workspace_bytes(dtype_code(self.m), self.fid, Q, T, N)
        if workspace_bytes is not None:
            need = min(need, int(workspace_bytes))
        self.ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        self.det = torch.from_numpy(identity_packed(f.n, Q)).to(self.device)
        self.err_rand = torch.empty(T, dtype=torch.float64, device=self.device)
        self.err_det = torch.empty(T, dtype=torch.float64, device=self.device)
        self.nf_rand = torch.empty(T, dtype=torch.uint8, device=self.device)
        self.nf_det = torch.empty(T, dtype=torch.uint8, device=self.device)

    def run(self, a, b, plans, with_det: bool = True, stream=None):
        """Enqueue one pass on ``stream`` (default: torch's current stream)."""
        torch = self.torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = _lib.load().rbc_error_trials_async(
            dtype_code(self.m), self.fid, self.Q, self.T, self.N,
            ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
            ctypes.c_void_p(plans.data_ptr()) if plans is not None else None,
            ctypes.c_void_p(self.det.data_ptr()) if with_det else None,
            ctypes.c_void_p(self.err_rand.data_ptr()), ctypes.c_void_p(self.err_det.data_ptr()),
            ctypes.c_void_p(self.nf_rand.data_ptr()), ctypes.c_void_p(self.nf_det.data_ptr()),
            ctypes.c_void_p(self.ws.data_ptr()), self.ws.numel(), ctypes.c_void_p(st.cuda_stream),
        )
        _lib.check(rc)
