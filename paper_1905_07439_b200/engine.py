"""Drop-in replacement for the reference engine ``randbc._engine``.

``apply_levels`` and ``leaf_matmul`` keep the reference signatures, argument
meaning, return values and exceptions (reference
``pkg/src/randbc/_engine.py:42-61`` and ``:117-149``) and run on the B200
through the C ABI of ``librbc.so`` (include/rbc.h).  ``install()`` assigns them
into ``randbc._engine``; every reference caller resolves the attribute at
call time (multiply.py:51,69,99; randomize.py:219,230,273,322), so the whole
reference library then multiplies on the GPU.

``apply_plans`` is the accelerator extension used by this package's own L2
mirror (``multiply``/``randomize``): for exact +-1 formulas it evaluates the
recursion straight from the randomization plans instead of from hatted
coefficient tables (same values; see csrc/kernels_plan.cu).

There is no CPU fallback anywhere in this module.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .precision import dtype_code, mode_of

__all__ = ["apply_levels", "leaf_matmul", "apply_plans", "pack_plans", "rel_errors", "install",
           "uninstall"]


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


def _as_mode_array(x, dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x), dtype=dtype)


class _PlanIndex:
    """Inverse map from hatted coefficient tables of one exact +-1 formula to
    the (perm, sign) pairs that produce them (reference randomize.py:163-178:
    uh[r,k,l] = u[r, pa(k), pb(l)] sa(k) sb(l), same for v with (p2, p3) and w
    with (p1, p3); the rescale factor of an exact formula is exactly 1)."""

    def __init__(self, fid, f):
        import itertools

        self.fid, self.n, self.R = fid, f.n, f.rank
        n = f.n
        perms = list(itertools.permutations(range(n)))
        signs = list(itertools.product((1.0, -1.0), repeat=n))
        self.maps = []
        for t in (f.u, f.v, f.w):
            d = {}
            for pa in perms:
                for pb in perms:
                    h = t[:, list(pa)][:, :, list(pb)]
                    for sa in signs:
                        for sb in signs:
                            key = (h * np.outer(sa, sb)[None]).astype(np.int8).tobytes()
                            d.setdefault(key, []).append((pa, pb, sa, sb))
            self.maps.append(d)

    def match(self, key):
        """Plan (perms (3, n), signs (3, n)) for one trial's int8 (u, v, w)
        row (3 * R * n * n entries), or None."""
        k = self.R * self.n * self.n
        cu, cv, cw = (self.maps[i].get(key[i * k:(i + 1) * k].tobytes()) for i in range(3))
        if not (cu and cv and cw):
            return None
        for p1, p2, s1, s2 in cu:
            for q2, p3, t2, s3 in cv:
                if q2 != p2 or t2 != s2:
                    continue
                for r1, r3, u1, u3 in cw:
                    if r1 == p1 and r3 == p3 and u1 == s1 and u3 == s3:
                        return np.array([p1, p2, p3], dtype=np.int64), np.array([s1, s2, s3])
        return None


_PLAN_INDEX = {}


def _plan_indexes(n, R):
    from .randomize import _known_formulas

    out = []
    for fid, f in _known_formulas():
        if f.n == n and f.rank == R:
            if fid not in _PLAN_INDEX:
                _PLAN_INDEX[fid] = _PlanIndex(fid, f)
            out.append(_PLAN_INDEX[fid])
    return out


def detect_plans(tabs):
    """If every level's tables are hatted tables of one known exact +-1
    formula, return (formula id, packed (Tp, Q, 40) plans); else None.
    RBC_DETECT_PLANS=0 turns recognition off (everything runs dense)."""
    import os

    if os.environ.get("RBC_DETECT_PLANS", "1") == "0":
        return None
    found = match_plans(tabs)
    if found is None:
        return None
    fid, perms, signs = found
    Tp, Q, _, n = perms.shape
    packed = pack_plans(n, perms.reshape(Tp * Q, 3, n), signs.reshape(Tp * Q, 3, n))
    return fid, packed.reshape(Tp, Q, -1)


def match_plans(tabs):
    """(formula id, perms (Tp, Q, 3, n), signs (Tp, Q, 3, n)) reproducing
    every level's (u, v, w) tables, or None.  The plan is unique only up to
    the formula's symmetries (always including the global sign flip s -> -s);
    any plan giving the same tables gives the same evaluation."""
    Q = len(tabs)
    n, R = tabs[0][0].shape[2], tabs[0][0].shape[1]
    if any(lv[0].shape[2] != n or lv[0].shape[1] != R for lv in tabs):
        return None
    Tp = max(lv[0].shape[0] for lv in tabs)
    # one int8 row per (level, trial); distinct rows are matched once each
    rows = []
    for u, v, w in tabs:
        flat = np.concatenate([t.reshape(t.shape[0], -1) for t in (u, v, w)], axis=1)
        f64 = flat.astype(np.float64)
        if not np.all((f64 == 0.0) | (f64 == 1.0) | (f64 == -1.0)):
            return None
        uniq, inv = np.unique(flat.astype(np.int8), axis=0, return_inverse=True)
        rows.append((uniq, inv.reshape(-1)))
    for idx in _plan_indexes(n, R):
        perms = np.zeros((Tp, Q, 3, n), dtype=np.int64)
        signs = np.zeros((Tp, Q, 3, n))
        ok = True
        for q, (uniq, inv) in enumerate(rows):
            up = np.zeros((len(uniq), 3, n), dtype=np.int64)
            us = np.zeros((len(uniq), 3, n))
            for j, key in enumerate(uniq):
                res = idx.match(key)
                if res is None:
                    ok = False
                    break
                up[j], us[j] = res
            if not ok:
                break
            perms[:, q], signs[:, q] = up[inv], us[inv]
        if ok:
            return idx.fid, perms, signs
    return None


def apply_levels(levels, a, b, mode, stats=None) -> np.ndarray:
    """Evaluate a blocked formula recursion (reference _engine.py:117-149).

    levels : sequence of (u, v, w), each (Tc, R, n, n) in the mode's dtype,
             Tc in {1, T}; levels[0] splits the full operands
    a, b   : (T0, s, s) mode-typed operands, T0 in {1, T}
    returns: (T, s, s) mode-typed array (a new host array)

    Tables that are signed permutations of a known exact +-1 formula (what the
    reference's L2 passes for Strassen / Laderman) are recognised and run on
    the plan-path kernels; anything else runs on the dense kernels.  Both give
    the reference's values.
    """
    m = mode_of(mode)
    if not levels:
        raise ValueError("need at least one level")
    dt = np.dtype(m.dtype)
    a = _as_mode_array(a, dt)
    b = _as_mode_array(b, dt)
    if a.ndim != 3 or b.ndim != 3 or a.shape != b.shape or a.shape[1] != a.shape[2]:
        raise ValueError("operands must be (T0, s, s) stacks of equal square matrices")
    T0, N, _ = a.shape
    tabs = []
    for lvl in levels:
        u, v, w = (_as_mode_array(t, dt) for t in lvl)
        if u.ndim != 4 or v.ndim != 4 or w.ndim != 4:
            raise ValueError("coefficient tables must have shape (Tc, R, n, n)")
        core = u.shape[1:]
        if v.shape[1:] != core or w.shape[1:] != core or core[1] != core[2]:
            raise ValueError("u, v, w of one level must share (R, n, n)")
        tabs.append([u, v, w])
    T = max([T0] + [t.shape[0] for lvl in tabs for t in lvl])
    for lvl in tabs:
        for k, t in enumerate(lvl):
            if t.shape[0] not in (1, T):
                raise ValueError("coefficient trial axis does not broadcast")
        tc = max(t.shape[0] for t in lvl)
        # one trial count per level on the C side: broadcast the odd ones out
        for k, t in enumerate(lvl):
            if t.shape[0] != tc:
                lvl[k] = np.ascontiguousarray(np.broadcast_to(t, (tc,) + t.shape[1:]))
    if T0 not in (1, T):
        raise ValueError("operand trial axis does not broadcast")
    Q = len(tabs)
    s, divisible = N, True
    for lvl in tabs:
        divisible = divisible and s % lvl[0].shape[2] == 0
        s //= lvl[0].shape[2]
    if divisible and N > 0 and T > 0:
        found = detect_plans(tabs)
        if found is not None:
            fid, packed = found
            return apply_plans(fid, Q, packed, a, b, mode, stats)
    n_arr = (ctypes.c_int32 * Q)(*[lvl[0].shape[2] for lvl in tabs])
    R_arr = (ctypes.c_int32 * Q)(*[lvl[0].shape[1] for lvl in tabs])
    Tc_arr = (ctypes.c_int64 * Q)(*[lvl[0].shape[0] for lvl in tabs])
    u_arr = (ctypes.c_void_p * Q)(*[lvl[0].ctypes.data for lvl in tabs])
    v_arr = (ctypes.c_void_p * Q)(*[lvl[1].ctypes.data for lvl in tabs])
    w_arr = (ctypes.c_void_p * Q)(*[lvl[2].ctypes.data for lvl in tabs])
    out = np.empty((T, N, N), dtype=dt)
    leaves = ctypes.c_uint64(0)
    lib = _lib.load()
    rc = lib.rbc_apply_levels(
        dtype_code(m), Q, n_arr, R_arr, Tc_arr, u_arr, v_arr, w_arr,
        T0, N, _ptr(a), _ptr(b), T, _ptr(out), ctypes.byref(leaves),
    )
    _lib.check(rc, overflow_msg=f"result left the {getattr(mode, 'kind', m.kind)} range")
    if stats is not None:
        stats["leaf_multiplies"] = stats.get("leaf_multiplies", 0) + int(leaves.value)
    return out


def leaf_matmul(x, y, mode) -> np.ndarray:
    """Batched product over the last two axes, sequential over the shared
    dimension (reference _engine.py:42-61)."""
    m = mode_of(mode)
    dt = np.dtype(m.dtype)
    x = np.asarray(x)
    y = np.asarray(y)
    shared = x.shape[-1]
    if y.shape[-2] != shared:
        raise ValueError("inner dimensions do not conform")
    lead = np.broadcast_shapes(x.shape[:-2], y.shape[:-2])
    M, N = x.shape[-2], y.shape[-1]
    shape = lead + (M, N)
    if shared == 0:
        return m.array(np.zeros(shape))
    batch = int(math.prod(lead))
    out = np.empty(shape, dtype=dt)
    if batch == 0 or M == 0 or N == 0:
        return out

    def flat(t, tail):
        t = _as_mode_array(t, dt)
        if t.shape[:-2] == lead:
            return t, tail
        if int(math.prod(t.shape[:-2])) == 1:
            return np.ascontiguousarray(t.reshape(t.shape[-2:])), 0
        return np.ascontiguousarray(np.broadcast_to(t, lead + t.shape[-2:])), tail

    xf, xs = flat(x, M * shared)
    yf, ys = flat(y, shared * N)
    rc = _lib.load().rbc_leaf_matmul(dtype_code(m), batch, xs, ys, M, shared, N,
                                     _ptr(xf), _ptr(yf), _ptr(out))
    _lib.check(rc)
    return out


def pack_plans(n: int, perms: np.ndarray, signs: np.ndarray) -> np.ndarray:
    """Pack (count, 3, n) perms / signs into the engine's 40-byte plan records."""
    perms = np.ascontiguousarray(perms, dtype=np.int64)
    signs = np.ascontiguousarray(signs, dtype=np.float64)
    if perms.shape != signs.shape or perms.ndim != 3 or perms.shape[1:] != (3, n):
        raise ValueError("perms and signs must both have shape (count, 3, n)")
    count = perms.shape[0]
    out = np.zeros((count, _lib.PLAN_BYTES), dtype=np.uint8)
    rc = _lib.load().rbc_pack_plans(n, count, _ptr(perms), _ptr(signs), _ptr(out))
    _lib.check(rc)
    return out


def apply_plans(formula_id: int, Q: int, packed: np.ndarray, a, b, mode, stats=None,
                return_flags: bool = False):
    """Q-level evaluation of an exact +-1 formula under packed plans.

    packed: (Tp, Q, 40) uint8 from ``pack_plans`` (Tp in {1, T});
    a, b  : (T0, N, N) mode-typed operands.
    Raises OverflowError like the reference when any output is non-finite,
    unless ``return_flags`` is set (then returns (out, per-trial flags)).
    """
    m = mode_of(mode)
    dt = np.dtype(m.dtype)
    a = _as_mode_array(a, dt)
    b = _as_mode_array(b, dt)
    if a.ndim != 3 or a.shape != b.shape or a.shape[1] != a.shape[2]:
        raise ValueError("operands must be (T0, s, s) stacks of equal square matrices")
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    if packed.ndim != 3 or packed.shape[1] != Q or packed.shape[2] != _lib.PLAN_BYTES:
        raise ValueError("packed plans must have shape (Tp, Q, 40)")
    T0, N, _ = a.shape
    Tp = packed.shape[0]
    T = max(T0, Tp)
    out = np.empty((T, N, N), dtype=dt)
    flags = np.zeros(max(T, 1), dtype=np.uint8)
    leaves = ctypes.c_uint64(0)
    rc = _lib.load().rbc_apply_plans(
        dtype_code(m), formula_id, Q, Tp, _ptr(packed), T0, N, _ptr(a), _ptr(b), T,
        _ptr(out), _ptr(flags), ctypes.byref(leaves),
    )
    if stats is not None and rc in (_lib.RBC_OK, _lib.RBC_EOVERFLOW):
        stats["leaf_multiplies"] = stats.get("leaf_multiplies", 0) + int(leaves.value)
    if return_flags and rc == _lib.RBC_EOVERFLOW:
        return out, flags[:T].astype(bool)
    _lib.check(rc, overflow_msg=f"result left the {getattr(mode, 'kind', m.kind)} range")
    return (out, flags[:T].astype(bool)) if return_flags else out


def _vp(t):
    """Device pointer of a torch tensor handed to the C ABI, which assumes
    dense row-major storage: a strided view would be read as garbage."""
    if not t.is_contiguous():
        raise ValueError("device tensors passed to librbc must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


class DeviceEngine:
    """Device-resident twin of apply_levels / apply_plans over torch CUDA
    tensors and one stream (no host copies, no synchronisation)."""

    def __init__(self, mode, device="cuda:0", stream=None):
        import torch

        self.torch = torch
        self.m = mode_of(mode)
        self.code = dtype_code(self.m)
        self.device = torch.device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._ws = None

    def _workspace(self, nbytes):
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = self.torch.empty(max(int(nbytes), 1), dtype=self.torch.uint8, device=self.device)
        return self._ws

    def apply_plans(self, fid, Q, packed, a, b, out, nonfinite):
        """packed (Tp, Q, 40) uint8, a/b (T0, N, N), out (T, N, N), nonfinite (T,) uint8."""
        T, N = out.shape[0], out.shape[-1]
        lib = _lib.load()
        ws = self._workspace(lib.rbc_plans_workspace_bytes(self.code, fid, Q, T, N))
        rc = lib.rbc_apply_plans_async(
            self.code, fid, Q, packed.shape[0], _vp(packed), a.shape[0], N, _vp(a), _vp(b), T,
            _vp(out), _vp(nonfinite), _vp(ws), ws.numel(), ctypes.c_void_p(self.stream.cuda_stream))
        _lib.check(rc)

    def apply_levels(self, levels, a, b, out, nonfinite):
        """levels: Q device triples (Tc, R, n, n)."""
        Q = len(levels)
        T, N = out.shape[0], out.shape[-1]
        n_arr = (ctypes.c_int32 * Q)(*[lv[0].shape[2] for lv in levels])
        R_arr = (ctypes.c_int32 * Q)(*[lv[0].shape[1] for lv in levels])
        Tc = (ctypes.c_int64 * Q)(*[lv[0].shape[0] for lv in levels])
        ptrs = [(ctypes.c_void_p * Q)(*[_vp(lv[k]).value for lv in levels]) for k in range(3)]
        lib = _lib.load()
        ws = self._workspace(lib.rbc_levels_workspace_bytes(self.code, Q, n_arr, R_arr, T, N))
        rc = lib.rbc_apply_levels_async(
            self.code, Q, n_arr, R_arr, Tc, ptrs[0], ptrs[1], ptrs[2], a.shape[0], N, _vp(a), _vp(b),
            T, _vp(out), _vp(nonfinite), _vp(ws), ws.numel(), ctypes.c_void_p(self.stream.cuda_stream))
        _lib.check(rc)

    def sum_trials(self, x, total):
        """total (N*N,) float64 += x[0] + ... + x[T-1], sequentially."""
        rc = _lib.load().rbc_sum_trials_async(self.code, x.shape[0], x.shape[-1], _vp(x), _vp(total),
                                              ctypes.c_void_p(self.stream.cuda_stream))
        _lib.check(rc)


def truth(A, B, mode, device="cuda:0") -> np.ndarray:
    """Binary64 inner-product truth of mode-typed operands (T, N, N) -> (T, N, N)
    float64, k ascending (reference experiments.py:251-254 with
    standard_multiply(Ad, Bd, DOUBLE)); C ABI rbc_truth_async."""
    import torch

    m = mode_of(mode)
    A = np.ascontiguousarray(A, dtype=m.dtype)
    B = np.ascontiguousarray(B, dtype=m.dtype)
    if A.ndim != 3 or A.shape != B.shape or A.shape[1] != A.shape[2]:
        raise ValueError("operands must be (T, N, N) stacks of equal square matrices")
    T, N, _ = A.shape
    dev = torch.device(device)
    a = torch.from_numpy(A).to(dev)
    b = torch.from_numpy(B).to(dev)
    ref = torch.empty((T, N, N), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev)
    rc = _lib.load().rbc_truth_async(dtype_code(m), T, N, _vp(a), _vp(b), _vp(ref),
                                     ctypes.c_void_p(st.cuda_stream))
    _lib.check(rc)
    return ref.cpu().numpy()


def rel_errors(results, ref, refnorm, mode) -> np.ndarray:
    """Per-trial relative Frobenius errors of a (T, N, N) mode-typed stack
    against the binary64 product ``ref`` -- the reference's
    ``experiments._rel_errors(results, ref, refnorm, mode)``
    (experiments.py:258-261), reduced on the device (C ABI rbc_rel_errors).

    ``refnorm`` is accepted for the reference's signature; the device computes
    ||ref||_F itself in binary64 (it differs from ``np.linalg.norm`` by an ulp
    at most, like one BLAS from another)."""
    del refnorm
    m = mode_of(mode)
    res = _as_mode_array(results, np.dtype(m.dtype))
    ref = np.ascontiguousarray(ref, dtype=np.float64)
    if res.ndim != 3 or ref.shape != res.shape[1:] or res.shape[1] != res.shape[2]:
        raise ValueError("results must be (T, N, N) and ref (N, N)")
    T, N, _ = res.shape
    err = np.empty(T, dtype=np.float64)
    rc = _lib.load().rbc_rel_errors(dtype_code(m), T, N, _ptr(res), _ptr(ref), 0, _ptr(err))
    _lib.check(rc)
    return err


_saved = {}
_saved_wide = []


def _install_wide() -> None:
    """Also route the reference's callers of the engine -- the L2 entry points
    of SURVEY §8 rows a9, a10, a12 and §8f row 2 -- to this package's mirrors,
    which hand plans to the device instead of hatted tables (no host hatting,
    no table recognition) and reduce the errors on the device."""
    import randbc.experiments as rexp  # noqa: PLC0415
    import randbc.multiply as rmul  # noqa: PLC0415
    import randbc.randomize as rrand  # noqa: PLC0415
    import randbc.rescale as rresc  # noqa: PLC0415

    from . import multiply, randomize, rescale  # noqa: PLC0415

    targets = {
        "recursive_randomized_apply_many": randomize.recursive_randomized_apply_many,
        "recursive_randomized_apply": randomize.recursive_randomized_apply,
        "randomized_apply": randomize.randomized_apply,
        "recursive_apply": multiply.recursive_apply,
        "rescaled_multiply": rescale.rescaled_multiply,
        "_rel_errors": rel_errors,
    }
    for mod in (rexp, rmul, rrand, rresc):
        for name, fn in targets.items():
            if hasattr(mod, name):
                _saved_wide.append((mod, name, getattr(mod, name)))
                setattr(mod, name, fn)


def install(module=None, wide: bool = False):
    """Route ``randbc._engine.apply_levels`` / ``leaf_matmul`` to the GPU.

    ``module`` defaults to ``randbc._engine`` (the reference must be
    importable).  Returns the module; ``uninstall`` restores the originals.

    ``wide=True`` additionally replaces the reference's L2 functions
    (``recursive_randomized_apply[_many]``, ``randomized_apply``,
    ``recursive_apply``, ``rescaled_multiply``) and
    ``experiments._rel_errors`` in every reference module that binds them, so
    a whole ``run_experiment`` keeps plans, scalings and error reductions on
    the device side of the C ABI.
    """
    if module is None:
        import randbc._engine as module  # noqa: PLC0415  (reference package)
    _saved[id(module)] = (module, module.apply_levels, module.leaf_matmul)
    module.apply_levels = apply_levels
    module.leaf_matmul = leaf_matmul
    if wide:
        _install_wide()
    return module


def uninstall(module=None) -> None:
    if module is None:
        import randbc._engine as module  # noqa: PLC0415
    saved = _saved.pop(id(module), None)
    if saved is not None:
        _, module.apply_levels, module.leaf_matmul = saved
    while _saved_wide:
        mod, name, fn = _saved_wide.pop()
        setattr(mod, name, fn)
