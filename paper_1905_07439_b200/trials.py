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


class ErrorTrialStream:
    """Host-buffer error trials as a stream of calls that overlap: ``submit``
    enqueues one call (rbc_error_trials_begin) and returns a ticket,
    ``result(ticket)`` waits for it (rbc_error_trials_end) and returns the same
    dict as :func:`error_trials`.  With the next call submitted before the
    previous result is taken, its operands are copied host->device while the
    previous call computes; at most two calls are in flight.

    A, B and packed plans are read asynchronously: pass pinned arrays (e.g.
    ``torch.from_numpy(x).pin_memory().numpy()``) and keep them unchanged
    until the call's ``result``.  Values are those of :func:`error_trials`."""

    def __init__(self, f, Q: int, mode, with_det: bool = True):
        self.m = mode_of(mode)
        self.fid = plan_formula_id(f)
        if self.fid is None:
            raise NotImplementedError("error trials support the exact +-1 formulas (plan path)")
        self.Q, self.n, self.with_det = Q, f.n, bool(with_det)
        self._live = {}

    def submit(self, A, B, packed=None, rplans=None) -> int:
        m = self.m
        A = np.ascontiguousarray(A, dtype=m.dtype)
        B = np.ascontiguousarray(B, dtype=m.dtype)
        T, N, _ = A.shape
        if packed is None and rplans is not None:
            packed = pack_recursive_plans(list(rplans), self.Q, self.n)
        if packed is not None:
            packed = np.ascontiguousarray(packed, dtype=np.uint8)
            if packed.shape != (T, self.Q, _lib.PLAN_BYTES):
                raise ValueError("packed plans must be (T, Q, 40)")
        res = _pinned_results(T)
        ticket = ctypes.c_int64(-1)
        rc = _lib.load().rbc_error_trials_begin(
            dtype_code(m), self.fid, self.Q, T, N, _vp(A), _vp(B),
            _vp(packed) if packed is not None else None, int(self.with_det),
            _vp(res[0]), _vp(res[1]), _vp(res[2]), _vp(res[3]), ctypes.byref(ticket))
        _lib.check(rc)
        self._live[ticket.value] = (res, packed is not None, (A, B, packed))
        return ticket.value

    def result(self, ticket: int):
        res, has_plans, _keep = self._live.pop(ticket)
        _lib.check(_lib.load().rbc_error_trials_end(ticket))
        out = {}
        if has_plans:
            out["err_rand"], out["nf_rand"] = res[0].copy(), res[2].astype(bool)
        if self.with_det:
            out["err_det"], out["nf_det"] = res[1].copy(), res[3].astype(bool)
        return out


def _pinned_results(T: int):
    """err_rand, err_det (float64) and nf_rand, nf_det (uint8) in pinned host
    memory, so that the result copies of a begun call are asynchronous."""
    import torch

    e = torch.full((2, max(1, T)), float("nan"), dtype=torch.float64).pin_memory().numpy()
    f = torch.zeros((2, max(1, T)), dtype=torch.uint8).pin_memory().numpy()
    return e[0][:T], e[1][:T], f[0][:T], f[1][:T]


def checkpoint_grid(total: int):
    """Running-average checkpoints 1..9, 10..90, ..., plus total
    (reference experiments.py:304-316)."""
    if total < 1:
        raise ValueError("total must be >= 1")
    pts = set()
    decade = 1
    while decade <= total:
        pts.update(k * decade for k in range(1, 10) if k * decade <= total)
        decade *= 10
    pts.add(total)
    return sorted(pts)


class DeviceAverageTrials:
    """Averaging trials on the device (config 3): per pair the binary64 truth,
    the deterministic product, G randomized products with per-plan errors and
    running-mean errors at ``checkpoint_grid(G)`` (reference
    experiments.py:264-296).  Any formula (dense coefficient tables)."""

    def __init__(self, f, Q: int, N: int, mode, P: int, G: int, device="cuda:0", checkpoints=None):
        import torch

        from .multiply import mode_tensors

        self.torch = torch
        self.f, self.Q, self.N, self.P, self.G = f, Q, N, P, G
        self.m = mode_of(mode)
        self.device = torch.device(device)
        self.cps = list(checkpoints) if checkpoints is not None else checkpoint_grid(G)
        self.n_arr = (ctypes.c_int32 * Q)(*([f.n] * Q))
        self.R_arr = (ctypes.c_int32 * Q)(*([f.rank] * Q))
        lib = _lib.load()
        need = lib.rbc_average_trials_workspace_bytes(dtype_code(self.m), Q, self.n_arr, self.R_arr, G, N)
        self.ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        det = mode_tensors(f, self.m)
        self.det = [torch.from_numpy(np.ascontiguousarray(t)).to(self.device) for t in det]
        self.err_rand = torch.empty(P * G, dtype=torch.float64, device=self.device)
        self.err_mean = torch.empty(P * len(self.cps), dtype=torch.float64, device=self.device)
        self.err_det = torch.empty(P, dtype=torch.float64, device=self.device)
        self.nf_rand = torch.empty(P * G, dtype=torch.uint8, device=self.device)
        self.nf_det = torch.empty(P, dtype=torch.uint8, device=self.device)

    def tables(self, rplans):
        """Per-level (P*G, R, n, n) hatted tables on the device."""
        from .randomize import plan_levels

        if len(rplans) != self.P * self.G:
            raise ValueError("need P*G recursive plans")
        out = []
        for q in range(self.Q):
            u, v, w = plan_levels(self.f, [rp.levels[q] for rp in rplans], self.m)
            out.append(tuple(self.torch.from_numpy(np.ascontiguousarray(t)).to(self.device)
                             for t in (u, v, w)))
        return out

    def capture(self, a, b, tables, with_det: bool = True):
        """One pass as a CUDA graph (see DeviceErrorTrials.capture)."""
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.graph(g, stream=s):
            self.run(a, b, tables, with_det, stream=s)
        torch.cuda.current_stream(self.device).wait_stream(s)
        return g

    def run(self, a, b, tables, with_det: bool = True, stream=None):
        torch = self.torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        Q = self.Q
        def vp(ts):
            if not all(t.is_contiguous() for t in ts):
                raise ValueError("coefficient tables must be contiguous (T, R, n, n) tensors")
            return (ctypes.c_void_p * Q)(*[t.data_ptr() for t in ts])

        u = vp([tb[0] for tb in tables])
        v = vp([tb[1] for tb in tables])
        w = vp([tb[2] for tb in tables])
        du = vp([self.det[0]] * Q) if with_det else None
        dv = vp([self.det[1]] * Q) if with_det else None
        dw = vp([self.det[2]] * Q) if with_det else None
        cps = (ctypes.c_int32 * len(self.cps))(*self.cps)
        rc = _lib.load().rbc_average_trials_async(
            dtype_code(self.m), Q, self.n_arr, self.R_arr, self.P, self.G, self.N,
            ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), u, v, w, du, dv, dw,
            len(self.cps), cps, ctypes.c_void_p(self.err_rand.data_ptr()),
            ctypes.c_void_p(self.err_mean.data_ptr()),
            ctypes.c_void_p(self.err_det.data_ptr()) if with_det else None,
            ctypes.c_void_p(self.nf_rand.data_ptr()),
            ctypes.c_void_p(self.nf_det.data_ptr()) if with_det else None,
            ctypes.c_void_p(self.ws.data_ptr()), self.ws.numel(), ctypes.c_void_p(st.cuda_stream),
        )
        _lib.check(rc)

    def results(self):
        return {
            "err_rand": self.err_rand.cpu().numpy().reshape(self.P, self.G),
            "err_mean": self.err_mean.cpu().numpy().reshape(self.P, len(self.cps)),
            "err_det": self.err_det.cpu().numpy(),
            "nf_rand": self.nf_rand.cpu().numpy().reshape(self.P, self.G).astype(bool),
            "checkpoints": list(self.cps),
        }


def average_trials(f, Q: int, A, B, mode, rplans, G: int, checkpoints=None, device="cuda:0"):
    """Host-buffer entry point for averaging trials: (P, N, N) operands and
    P*G recursive plans in; per-plan, running-mean and deterministic errors out."""
    import torch

    m = mode_of(mode)
    A = np.ascontiguousarray(A, dtype=m.dtype)
    B = np.ascontiguousarray(B, dtype=m.dtype)
    P, N, _ = A.shape
    runner = DeviceAverageTrials(f, Q, N, m, P, G, device=device, checkpoints=checkpoints)
    tables = runner.tables(list(rplans))
    a = torch.from_numpy(A).to(runner.device, non_blocking=True)
    b = torch.from_numpy(B).to(runner.device, non_blocking=True)
    runner.run(a, b, tables)
    torch.cuda.synchronize(runner.device)
    return runner.results()


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

    def capture(self, a, b, plans, with_det: bool = True):
        """Capture one pass (every launch of the truth, both products, the
        forked lanes and the errors) into a CUDA graph; ``graph.replay()``
        re-runs it on the same tensors without per-launch host overhead.
        Run the pass eagerly once first (kernel attributes are set on first
        use, outside capture)."""
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.graph(g, stream=s):
            self.run(a, b, plans, with_det, stream=s)
        torch.cuda.current_stream(self.device).wait_stream(s)
        return g

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


def run_trial_set(cfg, first: int, total: int, T_step: int, device="cuda:0", pipelined: bool = True,
                  runners=None):
    """Error trials of pairs first .. first+total-1 of a trial config, T_step
    pairs per pass, with fresh inputs: each pass's operand pairs are drawn on
    the GPU (rbc_matgen, bit-identical to the host draw, reference
    experiments.py:237-239), its plans drawn natively (experiments.py:242-245),
    the truth and both products run (experiments.py:248-261) and the per-trial
    errors copied back.  Returns (err_rand, err_det, nf_rand, nf_det) host
    arrays in pair order.

    ``pipelined``: pass s+1's inputs are drawn on a second stream into the other
    of two operand buffers while pass s computes -- the generator is integer /
    DP-issue work that co-issues with the truth's DFMAs and the leaves' packed
    FMAs, and its host half (tail samples) runs while the GPU
    is busy.  Values do not depend on the schedule.  ``runners``: optional
    dict reused across calls (keyed by pass size)."""
    import torch

    from .configs import make_pairs_device, packed_plans

    dev = torch.device(device)
    f = cfg.formula_obj()
    runners = {} if runners is None else runners
    chunks = [(p0, min(T_step, first + total - p0)) for p0 in range(first, first + total, T_step)]
    if not chunks:
        z = np.zeros(0)
        return z, z.copy(), np.zeros(0, np.uint8), np.zeros(0, np.uint8)
    tdt = {"double": torch.float64, "single": torch.float32, "half": torch.float16}[cfg.mode.kind]
    nbuf = 2 if pipelined and len(chunks) > 1 else 1
    bufs = [tuple(torch.empty((T_step, cfg.N, cfg.N), dtype=tdt, device=dev) for _ in range(2))
            for _ in range(nbuf)]
    main = torch.cuda.current_stream(dev)
    # high priority: the draw's CTAs take SM slots as the (much larger) compute
    # grids retire theirs, instead of queueing behind every pending CTA
    gen = torch.cuda.Stream(device=dev, priority=-1) if nbuf == 2 else main
    ready = [torch.cuda.Event() for _ in range(nbuf)]
    consumed = [torch.cuda.Event() for _ in range(nbuf)]
    host = torch.empty((len(chunks), 4, T_step), dtype=torch.float64).pin_memory()

    def draw(i):
        p0, cnt = chunks[i]
        slot = i % nbuf
        with torch.cuda.stream(gen):
            if i >= nbuf:
                gen.wait_event(consumed[slot])  # the pass that read this buffer is done
            a, b = make_pairs_device(cfg, p0, cnt, dev, out=tuple(t[:cnt] for t in bufs[slot]))
            ready[slot].record(gen)
        packed = packed_plans(cfg, [cfg.plan_key(p) for p in range(p0, p0 + cnt)])
        return a, b, torch.from_numpy(packed)

    nxt = draw(0)
    for i, (p0, cnt) in enumerate(chunks):
        a, b, pl = nxt
        slot = i % nbuf
        if cnt not in runners:
            runners[cnt] = DeviceErrorTrials(f, cfg.Q, cfg.N, cfg.mode, cnt, device=dev)
        r = runners[cnt]
        main.wait_event(ready[slot])
        r.run(a, b, pl.to(dev, non_blocking=True))
        consumed[slot].record(main)
        res = torch.stack([r.err_rand, r.err_det, r.nf_rand.to(torch.float64), r.nf_det.to(torch.float64)])
        host[i, :, :cnt].copy_(res, non_blocking=True)
        if i + 1 < len(chunks):
            nxt = draw(i + 1)  # overlaps pass i when pipelined
    torch.cuda.synchronize(dev)
    out = [np.concatenate([host[i, k, :cnt].numpy() for i, (_, cnt) in enumerate(chunks)])
           for k in range(4)]
    return out[0], out[1], out[2].astype(np.uint8), out[3].astype(np.uint8)


def run_average_set(cfg, first: int, total: int, P_step: int, device="cuda:0", pipelined: bool = True):
    """Averaging trials (reference experiments.py:264-296) of pairs
    first .. first+total-1 of an averaging config (plans_per_pair = G > 1),
    P_step pairs per pass, with fresh inputs: each pass's pairs are drawn on the
    GPU, its P*G plans drawn natively and hatted on the host (dense
    coefficient tables, the path of a formula that is not exact), then the
    truth, the deterministic product, the G randomized products, their errors
    and the running-mean errors run on the device.  Returns a dict of host
    arrays: err_rand (total, G), err_mean (total, checkpoints), err_det
    (total,), checkpoints.  ``pipelined``: the next pass's draw and tables are
    prepared (second stream, host) while a pass computes."""
    import torch

    from . import hostrng
    from .configs import ROLE_PLAN, make_pairs_device
    from .randomize import RandomizationPlan, RecursivePlan

    dev = torch.device(device)
    f = cfg.formula_obj()
    G = cfg.plans_per_pair
    chunks = [(p0, min(P_step, first + total - p0)) for p0 in range(first, first + total, P_step)]
    runners = {}
    tdt = {"double": torch.float64, "single": torch.float32, "half": torch.float16}[cfg.mode.kind]
    nbuf = 2 if pipelined and len(chunks) > 1 else 1
    bufs = [tuple(torch.empty((P_step, cfg.N, cfg.N), dtype=tdt, device=dev) for _ in range(2))
            for _ in range(nbuf)]
    main = torch.cuda.current_stream(dev)
    gen = torch.cuda.Stream(device=dev, priority=-1) if nbuf == 2 else main
    ready = [torch.cuda.Event() for _ in range(nbuf)]
    consumed = [torch.cuda.Event() for _ in range(nbuf)]

    def runner_for(cnt):
        if cnt not in runners:
            runners[cnt] = DeviceAverageTrials(f, cfg.Q, cfg.N, cfg.mode, cnt, G, device=dev)
        return runners[cnt]

    def prepare(i):
        p0, cnt = chunks[i]
        slot = i % nbuf
        keys = [cfg.plan_key(p, j) for p in range(p0, p0 + cnt) for j in range(1, G + 1)]
        perms, signs = hostrng.draw_plans(
            cfg.n, cfg.seed, [(ROLE_PLAN, t, q) for t in keys for q in range(cfg.Q)])
        perms = perms.reshape(len(keys), cfg.Q, 3, cfg.n)
        signs = signs.reshape(len(keys), cfg.Q, 3, cfg.n)
        rplans = [RecursivePlan(tuple(RandomizationPlan(signs[t, q], perms[t, q]) for q in range(cfg.Q)))
                  for t in range(len(keys))]
        with torch.cuda.stream(gen):
            if i >= nbuf:
                gen.wait_event(consumed[slot])
            a, b = make_pairs_device(cfg, p0, cnt, dev, out=tuple(t[:cnt] for t in bufs[slot]))
            tables = runner_for(cnt).tables(rplans)
            ready[slot].record(gen)
        return a, b, tables

    out = {"err_rand": [], "err_mean": [], "err_det": []}
    ncp = len(checkpoint_grid(G))
    pin = {"err_rand": torch.empty((P_step, G), dtype=torch.float64).pin_memory(),
           "err_mean": torch.empty((P_step, ncp), dtype=torch.float64).pin_memory(),
           "err_det": torch.empty(P_step, dtype=torch.float64).pin_memory()}
    pending = None
    nxt = prepare(0) if chunks else None
    for i, (p0, cnt) in enumerate(chunks):
        a, b, tables = nxt
        slot = i % nbuf
        r = runner_for(cnt)
        main.wait_event(ready[slot])
        if pending is not None:  # the runner's result buffers are reused by every pass
            for k, v in pending.items():
                out[k].append(v)
            pending = None
        r.run(a, b, tables)
        consumed[slot].record(main)
        res = {"err_rand": pin["err_rand"][:cnt], "err_mean": pin["err_mean"][:cnt],
               "err_det": pin["err_det"][:cnt]}
        res["err_rand"].copy_(r.err_rand.view(cnt, G), non_blocking=True)
        res["err_mean"].copy_(r.err_mean.view(cnt, len(r.cps)), non_blocking=True)
        res["err_det"].copy_(r.err_det, non_blocking=True)
        if i + 1 < len(chunks):
            nxt = prepare(i + 1)  # overlaps pass i when pipelined
        torch.cuda.current_stream(dev).synchronize()  # pass i done: its results are on the host
        pending = {k: v.numpy().copy() for k, v in res.items()}
    if pending is not None:
        for k, v in pending.items():
            out[k].append(v)
    cps = checkpoint_grid(G)
    return {"err_rand": np.concatenate(out["err_rand"]) if chunks else np.zeros((0, G)),
            "err_mean": np.concatenate(out["err_mean"]) if chunks else np.zeros((0, len(cps))),
            "err_det": np.concatenate(out["err_det"]) if chunks else np.zeros(0),
            "checkpoints": cps}
