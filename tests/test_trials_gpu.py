"""GPU: the error-trial pipeline (truth, products, relative errors) against
the CPU oracle on the config seed layout, host-buffer and device paths."""

import numpy as np
import pytest

from oracle import engine as oracle

pytestmark = pytest.mark.gpu


def _oracle_errors(cfg, f, A, B, rplans):
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.randomize import plan_levels

    out = {"err_det": [], "err_rand": [], "nf_det": [], "nf_rand": []}
    for t in range(A.shape[0]):
        ref = oracle.standard_multiply(A[t].astype(np.float64), B[t].astype(np.float64))
        for key, levels in (
            ("det", [mode_tensors(f, cfg.mode)] * cfg.Q),
            ("rand", [plan_levels(f, [rplans[t].levels[q]], cfg.mode) for q in range(cfg.Q)]),
        ):
            with np.errstate(all="ignore"):
                try:
                    C = oracle.apply_levels(levels, A[t][None], B[t][None], cfg.mode)
                    out["err_" + key].append(oracle.rel_errors(C, ref)[0])
                    out["nf_" + key].append(False)
                except OverflowError:
                    out["err_" + key].append(np.nan)
                    out["nf_" + key].append(True)
    return {k: np.array(v) for k, v in out.items()}


@pytest.mark.parametrize(
    "name,N,Q,T",
    [("c1", 64, 2, 5), ("c2", 81, 3, 4), ("c4", 64, 3, 4), ("c5", 128, 3, 2)],
)
def test_error_trials_match_oracle(name, N, Q, T):
    from dataclasses import replace

    from paper_1905_07439_b200.configs import get_config, make_pairs
    from paper_1905_07439_b200.trials import error_trials

    cfg = replace(get_config(name), N=N, Q=Q)
    f = cfg.formula_obj()
    A, B = make_pairs(cfg, 1, T)
    rplans = [cfg.plan(cfg.plan_key(p)) for p in range(1, T + 1)]
    got = error_trials(f, Q, A, B, cfg.mode, rplans=rplans)
    want = _oracle_errors(cfg, f, A, B, rplans)
    for key in ("det", "rand"):
        assert np.array_equal(got["nf_" + key], want["nf_" + key])
        ok = ~want["nf_" + key]
        np.testing.assert_allclose(got["err_" + key][ok], want["err_" + key][ok], rtol=1e-12, atol=0)


@pytest.mark.parametrize("label,N", [("f32", 243), ("f32", 256), ("f16", 200), ("f32", 37),
                                     ("f64", 260), ("f32", 520), ("f16", 640)])
def test_truth_bitwise(label, N):
    """The binary64 truth of narrow operands uses DFMA, which is exact here
    because every product of two widened f32/f16 values is exact in binary64:
    results must equal the sequential DMUL+DADD oracle bit for bit, including
    subnormal and large-magnitude inputs."""
    from paper_1905_07439_b200 import engine
    from paper_1905_07439_b200.precision import parse_precision

    mode = parse_precision(label)
    g = np.random.default_rng(N)
    A = g.standard_normal((3, N, N))
    B = g.standard_normal((3, N, N))
    tiny = 1e-40 if label == "f32" else 1e-7
    big = 1e30 if label == "f32" else 3e2
    A[0, :5, :5] *= tiny
    B[1, -5:, :] *= big
    A[2] = np.round(A[2] * 8) / 8  # heavy cancellation
    A, B = mode.array(A), mode.array(B)
    got = engine.truth(A, B, mode)
    for t in range(3):
        want = oracle.standard_multiply(A[t].astype(np.float64), B[t].astype(np.float64))
        assert got[t].tobytes() == want.tobytes()


@pytest.mark.parametrize("tile", ["0", "303"])
@pytest.mark.parametrize("shape", [(2, 130, 70, 257), (3, 128, 1, 128), (1, 300, 17, 140),
                                   (2, 129, 300, 131), (1, 515, 40, 600)])
def test_binary64_leaf_tiles_bitwise(shape, tile, monkeypatch):
    """binary64 leaves of 128 and up run on the binary64 tile kernels with
    DMUL + DADD (tile "303" forces the bulk-copy kernel at every size): ragged
    M/N (pad rows never stored), K tails shorter than a k tile, K = 1 (the
    initialising multiply only), broadcast operands."""
    monkeypatch.setenv("RBC_LEAF_TILE", tile)
    from paper_1905_07439_b200 import engine
    from paper_1905_07439_b200.precision import DOUBLE

    T, M, K, N = shape
    g = np.random.default_rng(M * K + N)
    x = g.standard_normal((T, M, K))
    y = g.standard_normal((T, K, N))
    x[0, :3, :] = -0.0  # products of -0 keep their sign on the first term
    got = engine.leaf_matmul(x, y, DOUBLE)
    want = oracle.leaf(x, y)
    assert got.tobytes() == want.tobytes()
    got_b = engine.leaf_matmul(x[:1], y, DOUBLE)  # x broadcast over the batch
    want_b = oracle.leaf(x[:1], y)
    assert got_b.tobytes() == want_b.tobytes()


def _same_bits_or_nan(got, want):
    """Bitwise equality, except that NaNs (inf - inf after an overflow) only
    need to be NaN in the same places: their sign/payload is not IEEE-defined
    and the reference raises OverflowError before any escapes (_engine.py:147)."""
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    assert got[~nan].tobytes() == want[~nan].tobytes()


@pytest.mark.parametrize("tile", ["0", "999"])
@pytest.mark.parametrize("shape", [(3, 128, 128, 128), (1, 256, 64, 136), (2, 130, 24, 200),
                                   (1, 128, 40, 128), (1, 128, 13, 128)])
def test_binary16_leaf_tiles_bitwise(shape, tile, monkeypatch):
    """binary16 leaves of 128 and up (config 4's leaves): the half2 tile
    kernels against the oracle's per-operation rounding, with ragged M/N, K
    tails (K not a multiple of the k tile; K = 13 falls back to the scalar
    loads), overflow to inf and signed zeros."""
    from paper_1905_07439_b200 import engine
    from paper_1905_07439_b200.precision import HALF

    monkeypatch.setenv("RBC_LEAF_TILE", tile)
    T, M, K, N = shape
    g = np.random.default_rng(M + 7 * K + N)
    x = HALF.array(g.standard_normal((T, M, K)) * 8)
    y = HALF.array(g.standard_normal((T, K, N)) * 8)
    x[0, :2, :] = -0.0
    x[0, 5, :] = 200.0  # row 5 overflows to +-inf
    with np.errstate(all="ignore"):
        got = engine.leaf_matmul(x, y, HALF)
        want = oracle.leaf(x, y)
    _same_bits_or_nan(got, want)


@pytest.mark.parametrize("tile", ["0", "999"])
@pytest.mark.parametrize("shape", [(3, 128, 128, 128), (1, 256, 64, 136), (2, 130, 24, 200),
                                   (4, 64, 64, 64), (1, 128, 13, 128), (2, 100, 36, 68)])
def test_binary32_leaf_tiles_bitwise(shape, tile, monkeypatch):
    """binary32 leaves (configs 1 and 5): the vector-load tile kernels against
    the oracle, with ragged M/N, K tails, a K that is not a multiple of 4
    (scalar fallback), overflow and signed zeros."""
    from paper_1905_07439_b200 import engine
    from paper_1905_07439_b200.precision import SINGLE

    monkeypatch.setenv("RBC_LEAF_TILE", tile)
    T, M, K, N = shape
    g = np.random.default_rng(M + 11 * K + N)
    x = SINGLE.array(g.standard_normal((T, M, K)))
    y = SINGLE.array(g.standard_normal((T, K, N)))
    x[0, :2, :] = -0.0
    x[0, 5, :] = 3e38  # row 5 overflows
    with np.errstate(all="ignore"):
        got = engine.leaf_matmul(x, y, SINGLE)
        want = oracle.leaf(x, y)
    _same_bits_or_nan(got, want)


@pytest.mark.parametrize("label", ["f64", "f32"])
@pytest.mark.parametrize("tile,T", [("0", 4099), ("205", 4099), ("0", 2048), ("0", 2051), ("0", 3553)])
def test_small_square_leaves_bitwise(label, tile, T, monkeypatch):
    """27x27 leaves in long batches (config 3's leaves) run on the warp-per-leaf
    ring kernel (tile "0": 9 x 3 outputs per lane, bulk-copy slots) or the
    single-shot shared-memory kernel ("205"): both equal the oracle; odd batches
    end the chunks ragged and put leaves at 8-byte offsets, 2048 is the
    smallest batch the ring kernel takes (its last CTA gets no leaf), 2051 and
    3553 leave CTAs with fewer leaves than consumer warps / a short last chunk."""
    from paper_1905_07439_b200 import engine
    from paper_1905_07439_b200.precision import parse_precision

    monkeypatch.setenv("RBC_LEAF_TILE", tile)
    mode = parse_precision(label)
    g = np.random.default_rng(27)
    x = mode.array(g.standard_normal((T, 27, 27)))
    y = mode.array(g.standard_normal((T, 27, 27)))
    x[7, :2, :] = -0.0
    got = engine.leaf_matmul(x, y, mode)
    want = oracle.leaf(x, y)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("label", ["f64", "f32"])
def test_ring_leaves_long_batch_equal_single_shot(label, monkeypatch):
    """The ring kernel's slot reuse on a config-3 sized batch (146,004 leaves:
    every slot is refilled about 60 times per CTA), three launches, against the
    single-shot kernel on the device and the oracle on a sample.  A release
    that lets the refill overtake loads in flight shows up here as a few wrong
    rows per launch."""
    import ctypes

    import torch

    from paper_1905_07439_b200 import _lib
    from paper_1905_07439_b200.precision import parse_precision

    _lib.require_device()
    lib = _lib.load()
    mode = parse_precision(label)
    code = {"f64": 0, "f32": 1}[label]
    dt = {"f64": torch.float64, "f32": torch.float32}[label]
    T = 12167 * 12
    gen = torch.Generator(device="cuda").manual_seed(27)
    x = torch.randn(T, 27, 27, device="cuda", dtype=dt, generator=gen)
    y = torch.randn(T, 27, 27, device="cuda", dtype=dt, generator=gen)

    def run(tile):
        monkeypatch.setenv("RBC_LEAF_TILE", tile)
        out = torch.full((T, 27, 27), float("nan"), device="cuda", dtype=dt)
        st = torch.cuda.current_stream()
        _lib.check(lib.rbc_leaf_matmul_async(code, code, T, 729, 729, 27, 27, 27,
                                             ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                             ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st.cuda_stream)))
        torch.cuda.synchronize()
        return out

    want = run("205")
    for _ in range(3):
        got = run("0")
        assert torch.equal(got.view(torch.uint8), want.view(torch.uint8))
    pick = [0, 1, 4098, T - 2, T - 1]
    ref = oracle.leaf(mode.array(x[pick].cpu().numpy()), mode.array(y[pick].cpu().numpy()))
    assert want[pick].cpu().numpy().tobytes() == ref.tobytes()


def test_device_runner_matches_host_call():
    import torch

    from paper_1905_07439_b200.configs import get_config, make_pairs
    from paper_1905_07439_b200.randomize import pack_recursive_plans
    from paper_1905_07439_b200.trials import DeviceErrorTrials, error_trials

    from dataclasses import replace

    cfg = replace(get_config("c2"), N=81, Q=3)
    f = cfg.formula_obj()
    T = 6
    A, B = make_pairs(cfg, 1, T)
    packed = pack_recursive_plans([cfg.plan(p) for p in range(1, T + 1)], cfg.Q, cfg.n)
    host = error_trials(f, cfg.Q, A, B, cfg.mode, packed=packed)
    dev = torch.device("cuda:0")
    # a small workspace forces several trial chunks: values must not change
    r = DeviceErrorTrials(f, cfg.Q, cfg.N, cfg.mode, T, device=dev, workspace_bytes=1)
    import ctypes  # noqa: F401

    from paper_1905_07439_b200 import _lib
    from paper_1905_07439_b200.precision import dtype_code

    one = _lib.load().rbc_error_trials_workspace_bytes(dtype_code(cfg.mode), r.fid, cfg.Q, 2, cfg.N)
    r.ws = torch.empty(one, dtype=torch.uint8, device=dev)
    r.run(torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), torch.from_numpy(packed).to(dev))
    torch.cuda.synchronize()
    assert np.array_equal(r.err_rand.cpu().numpy(), host["err_rand"])
    assert np.array_equal(r.err_det.cpu().numpy(), host["err_det"])


@pytest.mark.parametrize("name,N,Q,T", [("c1", 256, 2, 5), ("c2", 243, 4, 3), ("c5", 1024, 3, 2)])
def test_graph_replay_matches_eager(name, N, Q, T):
    """The error-trial step captured as one CUDA graph (forked lanes, the
    stream-ordered scratch of the binary64 truth) replays to the same
    errors as eager launches, on fresh inputs written between replays."""
    import torch
    from dataclasses import replace

    from paper_1905_07439_b200.configs import get_config, make_pairs
    from paper_1905_07439_b200.randomize import pack_recursive_plans
    from paper_1905_07439_b200.trials import DeviceErrorTrials

    cfg = replace(get_config(name), N=N, Q=Q)
    f = cfg.formula_obj()
    dev = torch.device("cuda:0")
    A, B = make_pairs(cfg, 1, 2 * T)
    packed = pack_recursive_plans([cfg.plan(p) for p in range(1, 2 * T + 1)], cfg.Q, cfg.n)
    r = DeviceErrorTrials(f, cfg.Q, cfg.N, cfg.mode, T, device=dev)
    a = torch.from_numpy(A[:T]).to(dev)
    b = torch.from_numpy(B[:T]).to(dev)
    pl = torch.from_numpy(packed[:T]).to(dev)
    r.run(a, b, pl)
    torch.cuda.synchronize()
    g = r.capture(a, b, pl)
    for sl in (slice(T, 2 * T), slice(0, T)):
        a.copy_(torch.from_numpy(A[sl]))
        b.copy_(torch.from_numpy(B[sl]))
        pl.copy_(torch.from_numpy(packed[sl]))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        got = (r.err_rand.cpu().numpy().copy(), r.err_det.cpu().numpy().copy())
        r.run(a, b, pl)
        torch.cuda.synchronize()
        assert np.array_equal(got[0], r.err_rand.cpu().numpy())
        assert np.array_equal(got[1], r.err_det.cpu().numpy())


@pytest.mark.parametrize("name,N,Q", [("c2", 81, 3), ("c1", 64, 2)])
def test_trial_set_pipelined_equals_serial_and_host_call(name, N, Q):
    """trials.run_trial_set (fresh pairs drawn on the GPU for every pass; the
    next pass's draw on a second stream while a pass computes) returns the
    same per-trial errors pipelined and unpipelined, equal to the host-buffer
    call on host-drawn pairs (ragged last pass)."""
    from dataclasses import replace

    from paper_1905_07439_b200.configs import get_config, make_pairs
    from paper_1905_07439_b200.randomize import pack_recursive_plans
    from paper_1905_07439_b200.trials import error_trials, run_trial_set

    cfg = replace(get_config(name), N=N, Q=Q)
    total, T_step = 10, 4
    runs = [run_trial_set(cfg, 3, total, T_step, "cuda:0", pipelined=p) for p in (True, False, True)]
    for r in runs[1:]:
        for got, want in zip(r, runs[0]):
            assert got.tobytes() == want.tobytes()
    A, B = make_pairs(cfg, 3, total)
    packed = pack_recursive_plans([cfg.plan(p) for p in range(3, 3 + total)], cfg.Q, cfg.n)
    host = error_trials(cfg.formula_obj(), cfg.Q, A, B, cfg.mode, packed=packed)
    assert np.array_equal(runs[0][0], host["err_rand"]) and np.array_equal(runs[0][1], host["err_det"])


def test_release_device_memory_then_host_call_again():
    """rbc_release_device_memory frees the host-call arena; the next host-buffer
    call allocates again and returns the same values."""
    import paper_1905_07439_b200 as rbc
    from paper_1905_07439_b200 import _lib, engine
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.precision import SINGLE

    _lib.require_device()
    g = np.random.default_rng(5)
    f = rbc.strassen_formula()
    levels = [mode_tensors(f, SINGLE)] * 2
    a = SINGLE.array(g.standard_normal((3, 16, 16)))
    b = SINGLE.array(g.standard_normal((3, 16, 16)))
    first = engine.apply_levels(levels, a, b, SINGLE)
    _lib.check(_lib.load().rbc_release_device_memory())
    _lib.check(_lib.load().rbc_release_device_memory())  # idempotent
    again = engine.apply_levels(levels, a, b, SINGLE)
    assert again.tobytes() == first.tobytes()


def _stream_case(T, N=81, Q=3, first=1):
    from dataclasses import replace

    import torch

    from paper_1905_07439_b200.configs import get_config, make_pairs
    from paper_1905_07439_b200.randomize import pack_recursive_plans

    cfg = replace(get_config("c2"), N=N, Q=Q)
    A, B = make_pairs(cfg, first, T)
    packed = pack_recursive_plans([cfg.plan(p) for p in range(first, first + T)], cfg.Q, cfg.n)
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()  # noqa: E731
    return cfg, pin(A), pin(B), pin(packed)


def test_error_trial_stream_overlapped_calls_equal_single_calls():
    """rbc_error_trials_begin / _end with two calls in flight: five steps of
    different pairs, a shape change in the middle (the layout is rebuilt after
    the calls in flight have drained) and another host-buffer API between a
    submit and its result; every step equals the synchronous call bitwise."""
    import paper_1905_07439_b200 as rbc
    from paper_1905_07439_b200 import _lib, engine
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.precision import SINGLE
    from paper_1905_07439_b200.trials import ErrorTrialStream, error_trials

    _lib.require_device()
    steps = [_stream_case(T, first=1 + 40 * i) for i, T in enumerate([24, 24, 24, 7, 7, 24])]
    cfg = steps[0][0]
    f = cfg.formula_obj()
    want = [error_trials(f, cfg.Q, A, B, cfg.mode, packed=P) for _, A, B, P in steps]
    st = ErrorTrialStream(f, cfg.Q, cfg.mode)
    got = [None] * len(steps)
    prev = None
    g = np.random.default_rng(3)
    x = SINGLE.array(g.standard_normal((2, 16, 16)))
    lv = [mode_tensors(rbc.strassen_formula(), SINGLE)] * 2
    for i, (_, A, B, P) in enumerate(steps):
        t = st.submit(A, B, packed=P)
        if i == 2:  # takes the arena: waits for the two calls in flight first
            engine.apply_levels(lv, x, x, SINGLE)
        if prev is not None:
            got[prev[0]] = st.result(prev[1])
        prev = (i, t)
    got[prev[0]] = st.result(prev[1])
    for w, h in zip(want, got):
        for key in ("err_rand", "err_det", "nf_rand", "nf_det"):
            assert np.array_equal(w[key], h[key], equal_nan=True), key


def test_error_trial_stream_limits():
    """A third call in flight is refused; an unknown ticket is refused; an
    empty call completes."""
    from paper_1905_07439_b200 import _lib
    from paper_1905_07439_b200.trials import ErrorTrialStream

    _lib.require_device()
    cfg, A, B, P = _stream_case(8)
    st = ErrorTrialStream(cfg.formula_obj(), cfg.Q, cfg.mode)
    t0, t1 = st.submit(A, B, packed=P), st.submit(A, B, packed=P)
    with pytest.raises(ValueError):
        st.submit(A, B, packed=P)
    r0, r1 = st.result(t0), st.result(t1)
    assert np.array_equal(r0["err_rand"], r1["err_rand"])
    assert _lib.load().rbc_error_trials_end(12345) != 0
    te = st.submit(A[:0], B[:0], packed=P[:0])
    assert st.result(te)["err_rand"].shape == (0,)
    # pageable operands (plain numpy): the copies are staged, the values the same
    tp = st.submit(np.array(A), np.array(B), packed=np.array(P))
    assert np.array_equal(st.result(tp)["err_rand"], r0["err_rand"])


@pytest.mark.parametrize("label", ["f64", "f32"])
@pytest.mark.parametrize("which", ["x", "y"])
def test_ring_leaves_broadcast_operand(label, which):
    """The ring kernel with a broadcast operand (batch stride 0): every slot
    copy of that operand reads the same 27 x 27 block."""
    from paper_1905_07439_b200 import engine
    from paper_1905_07439_b200.precision import parse_precision

    mode = parse_precision(label)
    g = np.random.default_rng(29)
    T = 2600
    x = mode.array(g.standard_normal((1 if which == "x" else T, 27, 27)))
    y = mode.array(g.standard_normal((1 if which == "y" else T, 27, 27)))
    got = engine.leaf_matmul(x, y, mode)
    want = oracle.leaf(np.broadcast_to(x, (T, 27, 27)), np.broadcast_to(y, (T, 27, 27)))
    assert got.shape == (T, 27, 27) and got.tobytes() == want.tobytes()
