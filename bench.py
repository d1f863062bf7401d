#!/usr/bin/env python
"""Benchmark of the randomized BC multiply hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A *step* is one pass of the hot path over one batch of synthetic input (the
config's seed layout), on every rank:

* error-trial configs (c1, c2, c4, c5): for each of the rank's T operand
  pairs, the binary64 truth, the deterministic BC product and its error, and
  the randomized BC product (fresh per-level signed permutations) and its
  error -- 2 BC products per pair;
* averaging config (c3): for each of the rank's P pairs, the truth, the
  deterministic product, G = 32 randomized products, their errors and the
  running-mean errors (reference experiments.py:264-296) -- G + 1 products
  per pair.

Default workload: BASELINE.json configs[1] ("c2": Laderman <3,3,3;23>, Q=4,
n=243, f32, Uniform[-1,1], 1000 pairs per rank).

value  : effective GFLOP/s = 2 n^3 x (BC products per step, all ranks) /
         step time; inputs resident in HBM; CUDA events on the launch stream;
         max over ranks
e2e    : the same through the public host-buffer API (error_trials /
         average_trials): pinned host operands + plans copied H2D and the
         per-trial errors copied D2H inside the timed region
roofline: the stage with the largest share of the timed region, from the
         engine's CUDA-event stage profiler (algorithmic bytes or flops per
         launch / average launch duration) against MEASURED_PEAKS.json (HBM)
         or profiles/fp_peaks.json (exact-order CUDA-core rates)
cpu_baseline: the CPU oracle (numpy restatement of the reference engine,
         oracle/) on a bounded sample of the same workload, rank 0, 1 core
--impl reference: the CPU oracle arm on all host cores (the reference is pure
         Python/numpy and cannot be compiled into oracle/_ref)

Multi-GPU: one process per GPU (torchrun), each rank owns its own block of
pairs (weak scaling); the only collectives are the MAX of the step times and
an all-gather of per-trial error statistics (a few KB, NCCL).
"""

from __future__ import annotations

import argparse
import contextlib
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

HBM_FALLBACK_GBS = 6650.0
FP32_NOMINAL_TFLOPS = 148 * 128 * 1.965e9 / 1e12  # FMUL+FADD per MAC: 1 flop/lane/clk
METRIC = "effective GFLOP/s (2n^3/time) of randomized BC matmul error trials"

# per config: pairs per rank per step (GPU), CPU sample (pairs, products per
# pair, subtree depth) -- depth d evaluates branch 0 of the top d levels only,
# i.e. 1/R^d of every product (used where one full CPU product takes minutes)
DEFAULTS = {
    "c1": dict(pairs=100, cpu=(100, 2, 0)),
    "c2": dict(pairs=1000, cpu=(20, 2, 0)),
    "c3": dict(pairs=4, cpu=(1, 3, 0)),
    "c4": dict(pairs=16, cpu=(1, 1, 1)),
    "c5": dict(pairs=2, cpu=(1, 1, 2)),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--trials", type=int, default=0, help="pairs per rank per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches in the timed region")
    return ap.parse_args()


# --------------------------------------------------------------- helpers ----
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class NvmlClocks:
    """NVML poller (5 ms) across the timed region: SM clock samples and the
    clock-event (throttle) reasons seen; falls back to nvidia-smi."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index: int):
        import threading

        import pynvml

        self.nv = pynvml
        pynvml.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [v for v in vis.split(",") if v.strip()]
            if index < len(ids) and ids[index].strip().isdigit():
                index = int(ids[index])
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.samples, self.mask = [], 0
        self.stop_ev = threading.Event()
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)

    def _reasons(self):
        nv = self.nv
        for name in ("nvmlDeviceGetCurrentClocksEventReasons", "nvmlDeviceGetCurrentClocksThrottleReasons"):
            fn = getattr(nv, name, None)
            if fn is not None:
                try:
                    return int(fn(self.h))
                except Exception:  # noqa: BLE001
                    continue
        return 0

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.mask |= self._reasons()
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def start(self):
        self.thread.start()

    def stop(self):
        self.stop_ev.set()
        self.thread.join(timeout=5)
        reasons = sorted(v for k, v in self.REASONS.items() if self.mask & k)
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": reasons,
            "samples": len(self.samples),
            "source": "nvml 5 ms poll over the timed region",
        }


def make_clocks(index: int):
    try:
        return NvmlClocks(index)
    except Exception:  # noqa: BLE001
        return Clocks(index)


class Clocks:
    """nvidia-smi sampler running across the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=10)
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                rows.append(parts)
        os.unlink(self.path)
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(mx) if mx else None,
            "reasons": reasons,
            "samples": len(rows),
        }


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", HBM_FALLBACK_GBS), "measured (MEASURED_PEAKS.json)"
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def fp_peaks():
    """Exact-order (FMUL+FADD, DMUL+DADD, HMUL2+HADD2) CUDA-core rates
    measured by tools/fp_peak.cu (profiles/fp_peaks.json)."""
    p = ROOT / "profiles" / "fp_peaks.json"
    if p.exists():
        return json.loads(p.read_text()), "measured (profiles/fp_peaks.json)"
    return {"f32_tflops": FP32_NOMINAL_TFLOPS, "f64_tflops": FP32_NOMINAL_TFLOPS / 2,
            "f16_tflops": FP32_NOMINAL_TFLOPS}, "nominal (half2 issues at half the FP32 rate)"


def ncu_traffic(stage: str, config: str):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(config, {}).get(stage)


def subtree_smem_bytes_per_launch(cfg, pairs: int) -> float:
    """Algorithmic shared-memory bytes of one fused two-level subtree launch:
    per CTA (level-q0 block, side s0 = M n^2, s1 = M n) the expansions write
    and re-read R s1^2 + R^2 M^2 elements per operand, the leaves read both
    operands and write the products, the contractions read and write back:
    6 R s1^2 + 6 R^2 M^2 element accesses.  CTAs per launch: pairs x R^(Q-2)."""
    import numpy as np

    n, R, Q = cfg.n, cfg.rank, cfg.Q
    M = cfg.N // n ** Q
    s1 = M * n
    e = np.dtype(cfg.mode.dtype).itemsize
    per_cta = (6 * R * s1 * s1 + 6 * R * R * M * M) * e
    return float(per_cta) * pairs * R ** (Q - 2)


def network_ops(formula: str):
    """(expand_u, expand_v, contract_w) add/sub counts per position of the
    generated plan-path networks (paper_1905_07439_b200/csrc/formulas_gen.cuh)."""
    import re

    src = (ROOT / "paper_1905_07439_b200" / "csrc" / "formulas_gen.cuh").read_text()
    name = {"laderman": "FLaderman", "laderman_noisy": "FLaderman", "strassen": "FStrassen"}[formula]
    i = src.index(f"struct {name}")
    j = src.find("\nstruct ", i + 10)
    body = src[i:j if j > 0 else len(src)]
    out = []
    for fn in ("expand_u", "expand_v", "contract_w"):
        a = body.index(f"static void {fn}(")
        b = body.index("\n  }\n", a)
        out.append(len(re.findall(r"O::(?:add|sub)\(", body[a:b])))
    return tuple(out)


def subtree_fp_ops_per_launch(cfg, pairs: int) -> float:
    """Algorithmic floating-point operations of one fused two-level subtree
    launch (level-q0 block of side s0 = M n^2, s1 = M n): both expansions of
    both operands (network adds per position), the R^2 leaf products
    (M^2 (2M - 1) each: multiplies plus adds, first term initialising) and
    both contractions.  Blocks per launch: pairs x R^(Q-2)."""
    n, R, Q = cfg.n, cfg.rank, cfg.Q
    M = cfg.N // n ** Q
    s1 = M * n
    u, v, w = network_ops(cfg.formula)
    per_block = (s1 * s1 * (u + v) + R * M * M * (u + v) + R * R * M * M * (2 * M - 1)
                 + R * M * M * w + s1 * s1 * w)
    return float(per_block) * pairs * R ** (Q - 2)


def smem_peak_gbs(sm_mhz):
    """Nominal shared-memory bandwidth: 128 B/clk/SM x 148 SMs x SM clock."""
    return 128.0 * 148 * (sm_mhz or 1965.0) * 1e6 / 1e9


def roofline(prof: dict, config: str, cfg=None, pairs=None, sm_max_mhz=None):
    if not prof:
        return None
    stage, agg = max(prof.items(), key=lambda kv: kv[1]["ms"])
    avg_s = agg["ms"] / agg["count"] / 1e3
    per_launch_bytes = agg["bytes"] / agg["count"]
    per_launch_flops = agg["flops"] / agg["count"]
    total_ms = sum(v["ms"] for v in prof.values())
    if stage == "subtree_fused" and cfg is not None:
        # the bottom two levels never touch HBM: the bound is the exact-order
        # CUDA-core FP pipe over the subtree's algorithmic operations (the
        # kernel is issue-bound: operand movement -- shuffles, shared memory,
        # plan signs -- shares the issue slots); smem and HBM views kept
        ops = subtree_fp_ops_per_launch(cfg, pairs)
        peaks, how = fp_peaks()
        key = {"double": "f64_tflops", "single": "f32_tflops", "half": "f16_tflops"}[cfg.mode.kind]
        peak = peaks[key]
        achieved = ops / avg_s / 1e12
        smem_b = subtree_smem_bytes_per_launch(cfg, pairs)
        smem_peak = smem_peak_gbs(sm_max_mhz)
        hbm_peak, hbm_how = measured_peaks()
        return {
            "bound": "cuda-core-" + key.split("_")[0] + "-exact-order", "kernel": stage,
            "achieved": round(achieved, 3), "peak": round(peak, 2), "peak_source": how,
            "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": ncu_traffic(stage, config),
            "algorithmic_fp_ops_per_launch": ops,
            "algorithmic_bytes_per_launch": per_launch_bytes,
            "hbm_view": {"achieved": round(per_launch_bytes / avg_s / 1e9, 2), "peak": hbm_peak,
                         "unit": "GB/s", "peak_source": hbm_how,
                         "frac": round(per_launch_bytes / avg_s / 1e9 / hbm_peak, 4)},
            "smem_view": {"achieved": round(smem_b / avg_s / 1e9, 2), "peak": round(smem_peak, 2),
                          "unit": "GB/s",
                          "peak_source": "nominal 128 B/clk/SM x 148 SMs x max SM clock",
                          "algorithmic_smem_bytes_per_launch": smem_b,
                          "note": "bytes a shared-memory-staged two-level subtree moves; the "
                                  "register-resident kernel keeps level q0+1 in registers",
                          "frac": round(smem_b / avg_s / 1e9 / smem_peak, 4)},
            "leaf_flops_per_launch": per_launch_flops, "avg_launch_ms": round(avg_s * 1e3, 5),
            "share_of_profiled_time": round(agg["ms"] / total_ms, 4) if total_ms else None,
            "stages": {k: {"count": v["count"], "ms": round(v["ms"], 4)} for k, v in prof.items()},
        }
    if stage.startswith(("leaf", "truth")):
        peaks, how = fp_peaks()
        key = {"leaf_f32": "f32_tflops", "leaf_f16": "f16_tflops"}.get(stage, "f64_tflops")
        achieved = per_launch_flops / avg_s / 1e12
        peak = peaks[key]
        bound, unit = ("cuda-core-" + key.split("_")[0] + "-exact-order"), "TFLOP/s"
        if stage == "truth_f64" and cfg is not None and cfg.mode.kind != "double":
            # narrow operands widened to binary64: products are exact, so the
            # truth runs as DFMA (bit-identical); measured DFMA pipe peak
            peak = peaks.get("dfma_f64_tflops", 2.0 * peaks["f64_tflops"])
            bound = "cuda-core-f64-dfma"
            how += " (dfma_f64_tflops)"
    else:
        peak, how = measured_peaks()
        achieved = per_launch_bytes / avg_s / 1e9
        bound, unit = "hbm", "GB/s"
    tr = ncu_traffic(stage, config)
    return {
        "bound": bound, "kernel": stage, "achieved": round(achieved, 2), "peak": round(peak, 2),
        "peak_source": how, "unit": unit, "frac": round(achieved / peak, 4),
        "traffic": tr, "algorithmic_bytes_per_launch": per_launch_bytes,
        "algorithmic_flops_per_launch": per_launch_flops, "avg_launch_ms": round(avg_s * 1e3, 5),
        "share_of_profiled_time": round(agg["ms"] / total_ms, 4) if total_ms else None,
        "stages": {k: {"count": v["count"], "ms": round(v["ms"], 4)} for k, v in prof.items()},
    }


# ------------------------------------------------------------ CPU oracle ----
def _cpu_job(job):
    """One CPU work unit through the oracle: pair p, products js (0 = the
    deterministic product, j >= 1 = randomized plan j), evaluated on branch 0
    of the top `depth` levels (depth 0 = the whole product).  Returns
    (effective flops, errors) -- errors only for depth 0."""
    cfg_name, p, js, depth = job
    import numpy as np

    from oracle import engine as oracle
    from paper_1905_07439_b200.configs import get_config
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.randomize import plan_levels

    cfg = get_config(cfg_name)
    f = cfg.formula_obj()
    A, B = cfg.pair(p)
    ref = oracle.standard_multiply(A.astype(np.float64), B.astype(np.float64)) if depth == 0 else None
    errs = []
    with np.errstate(all="ignore"):
        for j in js:
            if j == 0:
                levels = [mode_tensors(f, cfg.mode)] * cfg.Q
            else:
                rp = cfg.plan(cfg.plan_key(p, j) if cfg.plans_per_pair > 1 else cfg.plan_key(p))
                levels = [plan_levels(f, [rp.levels[q]], cfg.mode) for q in range(cfg.Q)]
            x = A[None, None]
            y = B[None, None]
            for q in range(depth):
                u, v, _ = levels[q]
                x = oracle.combine(x, u)[:, :1]
                y = oracle.combine(y, v)[:, :1]
            try:
                C = oracle.apply_levels(levels[depth:], x[:, 0], y[:, 0], cfg.mode)
                errs.append(float(oracle.rel_errors(C, ref)[0]) if ref is not None else None)
            except OverflowError:
                errs.append(float("nan"))
    flops = 2.0 * cfg.N ** 3 * len(js) / float(cfg.rank) ** depth
    return flops, errs


def run_cpu_jobs(jobs, workers: int):
    import concurrent.futures as cf

    t0 = time.perf_counter()
    if workers > 1:
        with cf.ProcessPoolExecutor(max_workers=workers) as ex:
            res = list(ex.map(_cpu_job, jobs))
    else:
        res = [_cpu_job(j) for j in jobs]
    return time.perf_counter() - t0, res


def cpu_sample_jobs(cfg, first_pair: int, count: int, per_pair: int, depth: int):
    if cfg.plans_per_pair > 1:
        js = list(range(per_pair))  # det + plans 1..per_pair-1
    else:
        js = [0, 1][:per_pair] if per_pair <= 2 else [0, 1]
        if per_pair == 1:
            js = [1]
    return [(cfg.name, p, js, depth) for p in range(first_pair, first_pair + count)]


def describe_sample(cfg, count, per_pair, depth, seconds, cores):
    what = f"{count} pair(s) x {per_pair} product(s)"
    if depth:
        what += (f", each product evaluated on branch 0 of its top {depth} level(s) "
                 f"(1/{cfg.rank}^{depth} of the work, credited as 2n^3/{cfg.rank}^{depth})")
    return (f"{what} through oracle/engine.py (numpy restatement of randbc._engine), "
            f"{cores} process(es), {seconds:.1f} s")


# ------------------------------------------------------------ reference ----
def run_reference(args):
    from paper_1905_07439_b200.configs import get_config

    world, rank, _ = dist_env()
    cfg = get_config(args.config)
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    _, per_pair, depth = DEFAULTS[cfg.name]["cpu"]
    p = 1
    for _ in range(args.warmup):
        run_cpu_jobs(cpu_sample_jobs(cfg, p, cores, per_pair, depth), cores)
        p += cores
    total_s, total_flops = 0.0, 0.0
    for _ in range(args.steps):
        dt, res = run_cpu_jobs(cpu_sample_jobs(cfg, p, cores, per_pair, depth), cores)
        total_s += dt
        total_flops += sum(r[0] for r in res)
        p += cores
    ms = total_s / args.steps * 1e3
    value = total_flops / total_s / 1e9
    line = {
        "metric": METRIC, "impl": "reference", "value": round(value, 5), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg.mode.label,
        "data": "synthetic (seeded, reference seed layout)",
        "config": {"workload": cfg.name, "desc": cfg.note, "jobs_per_step": cores},
        "cpu_baseline": {
            "value": round(value, 5), "unit": "GFLOP/s", "cores": cores, "kind": "port",
            "sample": describe_sample(cfg, cores, per_pair, depth, ms / 1e3, cores) + " per step",
        },
        "e2e": {"value": round(value, 5), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ ours ----
@contextlib.contextmanager
def no_gc():
    """The host-buffer calls are timed by wall clock: a full collection of the
    harness's own Python objects (plans, records) inside the timed loop is a
    harness artefact (seen as 20-100 ms outliers), so collect first and pause
    the collector while timing."""
    import gc

    gc.collect()
    was = gc.isenabled()
    gc.disable()
    try:
        yield
    finally:
        if was:
            gc.enable()


class ErrorTrialWorkload:
    """c1, c2, c4, c5: 2 products per pair (plan path, packed plans)."""

    def __init__(self, cfg, pair_ids, A, B, dev, torch):
        from paper_1905_07439_b200.randomize import pack_recursive_plans
        from paper_1905_07439_b200.trials import DeviceErrorTrials

        self.cfg, self.torch = cfg, torch
        self.f = cfg.formula_obj()
        self.A, self.B = A, B
        self.packed = pack_recursive_plans([cfg.plan(cfg.plan_key(p)) for p in pair_ids], cfg.Q, cfg.n)
        self.a = torch.from_numpy(A).to(dev)
        self.b = torch.from_numpy(B).to(dev)
        self.pl = torch.from_numpy(self.packed).to(dev)
        self.runner = DeviceErrorTrials(self.f, cfg.Q, cfg.N, cfg.mode, len(pair_ids), device=dev)
        self.products = 2 * len(pair_ids)

    def run(self, stream):
        self.runner.run(self.a, self.b, self.pl, stream=stream)

    def capture(self):
        """The step as one CUDA graph (None: not capturable here)."""
        return self.runner.capture(self.a, self.b, self.pl)

    def results(self):
        r = self.runner
        return (r.err_rand.cpu().numpy(), r.err_det.cpu().numpy(),
                r.nf_rand.cpu().numpy().astype(bool), r.nf_det.cpu().numpy().astype(bool))

    def e2e(self, steps, warmup=3):
        """Public host-buffer call (rbc_error_trials) on pinned buffers; the
        first call is checked against the device-resident errors, then
        `warmup` untimed calls, then `steps` timed ones."""
        import numpy as np

        from paper_1905_07439_b200.trials import error_trials

        torch = self.torch
        A_pin = torch.from_numpy(self.A).pin_memory()
        B_pin = torch.from_numpy(self.B).pin_memory()
        P_pin = torch.from_numpy(self.packed).pin_memory()
        args = (self.f, self.cfg.Q, A_pin.numpy(), B_pin.numpy(), self.cfg.mode)
        res = error_trials(*args, packed=P_pin.numpy())
        err_r, err_d, _, _ = self.results()
        if not (np.array_equal(res["err_rand"], err_r, equal_nan=True)
                and np.array_equal(res["err_det"], err_d, equal_nan=True)):
            raise SystemExit("e2e errors differ from the device-resident run")
        pn = P_pin.numpy()
        for _ in range(max(0, warmup - 1)):
            error_trials(*args, packed=pn)
        self.e2e_calls = []
        with no_gc():
            t0 = time.perf_counter()
            for _ in range(steps):
                t1 = time.perf_counter()
                error_trials(*args, packed=pn)
                self.e2e_calls.append((time.perf_counter() - t1) * 1e3)
            ms = (time.perf_counter() - t0) / steps * 1e3
        h2d = self.A.nbytes + self.B.nbytes + self.packed.nbytes
        d2h = 2 * len(err_r) * 9
        return ms, h2d, d2h


class AverageWorkload:
    """c3: per pair truth + deterministic + G randomized products + running mean."""

    def __init__(self, cfg, pair_ids, A, B, dev, torch):
        from paper_1905_07439_b200.trials import DeviceAverageTrials

        self.cfg, self.torch = cfg, torch
        self.f = cfg.formula_obj()
        self.A, self.B = A, B
        G = cfg.plans_per_pair
        self.G = G
        self.rplans = [cfg.plan(cfg.plan_key(p, j)) for p in pair_ids for j in range(1, G + 1)]
        self.runner = DeviceAverageTrials(self.f, cfg.Q, cfg.N, cfg.mode, len(pair_ids), G, device=dev)
        self.tables = self.runner.tables(self.rplans)
        self.a = torch.from_numpy(A).to(dev)
        self.b = torch.from_numpy(B).to(dev)
        self.products = (G + 1) * len(pair_ids)

    def run(self, stream):
        self.runner.run(self.a, self.b, self.tables, stream=stream)

    def capture(self):
        return self.runner.capture(self.a, self.b, self.tables)

    def results(self):
        r = self.runner.results()
        nf_d = self.runner.nf_det.cpu().numpy().astype(bool)
        return (r["err_rand"].ravel(), r["err_det"], r["nf_rand"].ravel(), nf_d)

    def mean_errors(self):
        return self.runner.results()["err_mean"]

    def e2e(self, steps, warmup=3):
        """Public host-buffer call (average_trials): hatted tables built from the
        plans, operands and tables copied H2D, errors copied back, per step
        (first call checked, `warmup` - 1 more untimed)."""
        import numpy as np

        from paper_1905_07439_b200.trials import average_trials

        torch = self.torch
        A_pin = torch.from_numpy(self.A).pin_memory().numpy()
        B_pin = torch.from_numpy(self.B).pin_memory().numpy()
        args = (self.f, self.cfg.Q, A_pin, B_pin, self.cfg.mode, self.rplans, self.G)
        res = average_trials(*args)
        err_r, err_d, _, _ = self.results()
        if not np.array_equal(res["err_rand"].ravel(), err_r, equal_nan=True):
            raise SystemExit("e2e errors differ from the device-resident run")
        for _ in range(max(0, warmup - 1)):
            average_trials(*args)
        with no_gc():
            t0 = time.perf_counter()
            for _ in range(steps):
                average_trials(*args)
            ms = (time.perf_counter() - t0) / steps * 1e3
        es = np.dtype(self.cfg.mode.dtype).itemsize
        h2d = self.A.nbytes + self.B.nbytes + sum(
            3 * len(self.rplans) * self.cfg.rank * self.cfg.n ** 2 * es for _ in range(self.cfg.Q))
        d2h = (len(self.rplans) + len(self.runner.cps) * len(self.A) + len(self.A)) * 8
        return ms, h2d, d2h


def device_inputs(cfg, first, T, A, B, host_s, workers):
    """Informational: the same operand pairs drawn on the GPU (rbc_matgen,
    SURVEY §8f rank 4) -- time and bitwise agreement with the host draw that
    feeds the timed region."""
    import torch

    from paper_1905_07439_b200.configs import make_pairs_device

    make_pairs_device(cfg, first, min(T, 2))  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dA, dB = make_pairs_device(cfg, first, T)
    torch.cuda.synchronize()
    dev_s = time.perf_counter() - t0
    same = (dA.cpu().numpy().tobytes() == A.tobytes() and dB.cpu().numpy().tobytes() == B.tobytes())
    del dA, dB
    return {"kind": cfg.kind, "device_matgen_ms": round(dev_s * 1e3, 2),
            "host_numpy_ms": round(host_s * 1e3, 1), "host_workers": workers,
            "bitwise_equal": same}


def run_ours(args):
    import numpy as np
    import torch

    from paper_1905_07439_b200 import _lib, distributed
    from paper_1905_07439_b200.configs import get_config, make_pairs

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        dist = None
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    _lib.require_device()

    cfg = get_config(args.config)
    T = args.trials or DEFAULTS[cfg.name]["pairs"]
    first, _ = distributed.shard(rank, world, T)
    pair_ids = distributed.pair_ids(rank, world, T)
    workers = min(32, max(1, (os.cpu_count() or 2) // max(1, world)))
    t_host = time.perf_counter()
    A, B = make_pairs(cfg, first, T, workers=workers)
    t_host = time.perf_counter() - t_host
    inputs = device_inputs(cfg, first, T, A, B, t_host, workers)
    kind = AverageWorkload if cfg.plans_per_pair > 1 else ErrorTrialWorkload
    wl = kind(cfg, pair_ids, A, B, dev, torch)
    stream = torch.cuda.Stream(device=dev)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        wl.run(stream)
    torch.cuda.synchronize()
    # the step as a CUDA graph (error-trial workloads): replays skip the
    # per-launch host work; the stage profiler then runs on a separate
    # eager pass below (events cannot be timed inside replays)
    graph, graph_note = None, "eager launches"
    if not args.no_graph and hasattr(wl, "capture"):
        try:
            with torch.cuda.stream(stream):
                graph = wl.capture()
            for _ in range(2):
                graph.replay()
            torch.cuda.synchronize()
            graph_note = "CUDA graph replay (one graph per step)"
        except Exception as exc:  # noqa: BLE001 -- report and fall back to eager
            graph, graph_note = None, f"eager launches (graph capture failed: {exc})"
            torch.cuda.synchronize()
    barrier()
    clocks = make_clocks(local)
    clocks.start()
    _lib.profile_enable(graph is None)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if graph is not None:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                graph.replay()
            ev1.record(stream)
    else:
        ev0.record(stream)
        for _ in range(args.steps):
            wl.run(stream)
        ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    if graph is not None:  # stage profile from an eager pass of the same steps
        _lib.profile_enable(True)
        for _ in range(args.steps):
            wl.run(stream)
        torch.cuda.synchronize()
    prof = _lib.profile_summary()
    _lib.profile_enable(False)
    launches = sum(v["count"] for v in prof.values())
    dev_ms = ev0.elapsed_time(ev1) / args.steps
    err_r, err_d, nf_r, nf_d = wl.results()

    e2e = None
    if not args.no_e2e:
        barrier()
        e2e = wl.e2e(args.steps, args.warmup)

    tmax = distributed.max_over_ranks([dev_ms, e2e[0] if e2e else 0.0], device=dev)
    dev_ms = float(tmax[0])
    allerr = distributed.gather_trials(
        np.stack([err_r, nf_r.astype(np.float64)]), device=dev)
    alldet = distributed.gather_trials(np.stack([err_d, nf_d.astype(np.float64)]), device=dev)

    flops_step = 2.0 * cfg.N ** 3 * wl.products * world
    value = flops_step / (dev_ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dev_ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg.mode.label,
        "data": "synthetic (seeded pairs and plans, reference seed layout; no dataset)",
        "trials_per_s": round(T * world / (dev_ms / 1e3), 3),
        "products_per_s": round(wl.products * world / (dev_ms / 1e3), 3),
        "config": {
            "workload": cfg.name, "desc": cfg.note, "formula": cfg.formula, "Q": cfg.Q,
            "n": cfg.N, "pairs_per_rank": T, "products_per_step_per_rank": wl.products,
            "parallelism": f"trial-sharded x{world}",
            "l2": f"per-step operands {A.nbytes * 2 / 1e6:.0f} MB + binary64 truth "
                  f"{min(T, 1 if cfg.plans_per_pair > 1 else T) * cfg.N ** 2 * 8 / 1e6:.0f} MB and "
                  "BC intermediates stream through HBM; the level working sets exceed the 126 MB L2 "
                  "at these batch sizes, so no explicit flush is used",
        },
        "gpu_launches": launches,
        "launch_mode": graph_note,
        "inputs": inputs,
        "clocks": clk,
        "roofline": roofline(prof, cfg.name, cfg, T, clk.get("sm_max_mhz")),
        "errors": distributed.trial_stats(allerr[0], alldet[0], allerr[1] > 0, alldet[1] > 0),
    }
    if hasattr(wl, "mean_errors"):
        me = wl.mean_errors()
        line["errors"]["running_mean_at_G"] = {
            "mean": float(np.nanmean(me[:, -1])), "checkpoints": wl.runner.cps}
    if e2e is not None:
        e2e_ms = float(tmax[1])
        line["e2e"] = {"value": round(flops_step / (e2e_ms / 1e3) / 1e9, 3), "unit": "GFLOP/s",
                       "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": int(e2e[1]),
                       "d2h_bytes_per_step": int(e2e[2])}
        calls = getattr(wl, "e2e_calls", None)
        if calls:
            line["e2e"]["ms_per_call"] = [round(c, 2) for c in calls]

    if rank == 0 and world == 1 and not args.no_cpu:
        count, per_pair, depth = DEFAULTS[cfg.name]["cpu"]
        jobs = cpu_sample_jobs(cfg, first, count, per_pair, depth)
        dt, res = run_cpu_jobs(jobs, 1)
        cpu_val = sum(r[0] for r in res) / dt / 1e9
        agree = None
        if depth == 0 and cfg.plans_per_pair == 1 and per_pair == 2:
            got = np.stack([err_d[:count], err_r[:count]], axis=1)
            want = np.array([r[1] for r in res], dtype=np.float64)
            agree = bool(np.allclose(got, want, rtol=1e-10, atol=0, equal_nan=True))
        line["cpu_baseline"] = {
            "value": round(cpu_val, 6), "unit": "GFLOP/s", "cores": 1, "kind": "port",
            "sample": describe_sample(cfg, count, per_pair, depth, dt, 1),
            "errors_agree_with_gpu": agree,
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
