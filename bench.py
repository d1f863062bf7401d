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
    ap.add_argument("--config", default="c5")
    ap.add_argument("--trials", type=int, default=0, help="pairs per rank per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches in the timed region")
    ap.add_argument("--no-tts", action="store_true", help="skip the time-to-solution run")
    ap.add_argument("--no-dropin", action="store_true", help="skip the drop-in s2-variants run")
    ap.add_argument("--dump-errors", default="", help="rank 0 writes the gathered per-trial errors (npz)")
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
    measured by tools/fp_peak.cu (profiles/fp_peaks.json).  The binary32
    denominator is the larger of the scalar (FMUL+FADD) and packed
    (FFMA2+FADD2) exact-order rates: the leaf kernels issue packed pairs."""
    p = ROOT / "profiles" / "fp_peaks.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["f32_tflops"] = max(d["f32_tflops"], d.get("f32x2_tflops", 0.0))
        return d, "measured (profiles/fp_peaks.json; binary32: max of FMUL+FADD, FFMA2+FADD2)"
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
    note = None
    if stage == "truth_f64" and tr and tr > 4 * per_launch_bytes:
        note = ("the binary64 truth streams its widened Y panels once per tile row (about 0.9 TB/s, "
                "14% of HBM) and is bound by the DFMA pipe, not by that traffic: rasters that share "
                "panels in L2 cut the reads 3.2x and ran 0.4-3% slower (DESIGN 4.1, "
                "profiles/r02/experiments/truth_raster_groups.txt)")
    return {
        "bound": bound, "kernel": stage, "achieved": round(achieved, 2), "peak": round(peak, 2),
        "peak_source": how, "unit": unit, "frac": round(achieved / peak, 4),
        "traffic": tr, "traffic_note": note, "algorithmic_bytes_per_launch": per_launch_bytes,
        "algorithmic_flops_per_launch": per_launch_flops, "avg_launch_ms": round(avg_s * 1e3, 5),
        "share_of_profiled_time": round(agg["ms"] / total_ms, 4) if total_ms else None,
        "stages": {k: {"count": v["count"], "ms": round(v["ms"], 4)} for k, v in prof.items()},
    }


# --------------------------------------------------------------- CPU side ----
REF_DIR = ROOT / "baseline" / "_ref"


def reference_available() -> bool:
    return (REF_DIR / "randbc" / "_engine.py").exists()


def reference_modules():
    """The unmodified reference package (baseline/_ref, installed by
    tools/reference_install.py from /root/reference/pkg)."""
    import types

    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import randbc._engine
    import randbc.experiments
    import randbc.formula
    import randbc.matgen
    import randbc.multiply
    import randbc.precision
    import randbc.randomize
    import randbc.rng

    return types.SimpleNamespace(engine=randbc._engine, experiments=randbc.experiments,
                                 formula=randbc.formula, matgen=randbc.matgen,
                                 multiply=randbc.multiply, precision=randbc.precision,
                                 randomize=randbc.randomize, rng=randbc.rng)


def cpu_kind() -> str:
    """'reference' when the unmodified reference is installed, else 'port'
    (oracle/engine.py, the numpy restatement of randbc._engine)."""
    return "reference" if reference_available() else "port"


class CpuJob:
    """One CPU work unit: pair p, products js (0 = the deterministic product,
    j >= 1 = randomized plan j), each evaluated on branch 0 of its top
    `depth` levels (depth 0 = the whole product; depth d = the sub-product of
    branch 0, 1/R^d of the work, credited as 2n^3/R^d), through the
    unmodified reference (`impl` 'reference') or the oracle port ('port').

    prepare(): inputs, plans, hatted tables and (depth 0) the binary64 truth
    -- untimed; compute(): the BC products only -- the timed part."""

    def __init__(self, cfg_name, p, js, depth, impl):
        self.cfg_name, self.p, self.js, self.depth, self.impl = cfg_name, p, tuple(js), depth, impl

    def prepare(self):
        import numpy as np

        from paper_1905_07439_b200.configs import get_config
        from paper_1905_07439_b200.precision import HALF

        cfg = self.cfg = get_config(self.cfg_name)
        fo = cfg.formula_obj()  # coefficient data (c3: builder noise on every entry)
        if self.impl == "reference":
            R = self.R = reference_modules()
            self.mode = {"double": R.precision.DOUBLE, "single": R.precision.SINGLE}.get(
                cfg.mode.kind, HALF)  # binary16: the duck-typed builder mode
            self.f = R.formula.BilinearFormula(fo.u, fo.v, fo.w)
            mseed = R.rng.derive_seed(cfg.seed, R.rng.ROLE_MATRIX, self.p,
                                      _kind_index(R, cfg.kind))
            A64, B64 = _ref_generate(R, cfg.kind, cfg.N, mseed)
            draw = lambda key: R.randomize.RecursivePlan(tuple(  # noqa: E731
                R.randomize.draw_plan(cfg.n, R.rng.derive_rng(cfg.seed, R.rng.ROLE_PLAN, key, q))
                for q in range(cfg.Q)))
            det_levels = lambda: [R.multiply.mode_tensors(self.f, self.mode)] * cfg.Q  # noqa: E731
            plan_levels = lambda rp: [R.randomize._plan_levels(self.f, [rp.levels[q]], self.mode)  # noqa: E731
                                      for q in range(cfg.Q)]
        else:
            from paper_1905_07439_b200.multiply import mode_tensors
            from paper_1905_07439_b200.randomize import plan_levels as ours_plan_levels

            self.mode, self.f = cfg.mode, fo
            A64 = B64 = None
            draw = cfg.plan
            det_levels = lambda: [mode_tensors(fo, cfg.mode)] * cfg.Q  # noqa: E731
            plan_levels = lambda rp: [ours_plan_levels(fo, [rp.levels[q]], cfg.mode)  # noqa: E731
                                      for q in range(cfg.Q)]
        if A64 is not None:
            self.A, self.B = self.mode.array(A64), self.mode.array(B64)
        else:
            self.A, self.B = cfg.pair(self.p)
        self.levels = []
        for j in self.js:
            if j == 0:
                self.levels.append(det_levels())
            else:
                key = cfg.plan_key(self.p, j) if cfg.plans_per_pair > 1 else cfg.plan_key(self.p)
                self.levels.append(plan_levels(draw(key)))
        self.ref = None
        if self.depth == 0:
            Ad = self.A.astype(np.float64)
            Bd = self.B.astype(np.float64)
            if self.impl == "reference":
                self.ref = self.R.multiply.standard_multiply(Ad, Bd, self.R.precision.DOUBLE)
            else:
                from oracle import engine as oracle

                self.ref = oracle.standard_multiply(Ad, Bd)
        return self

    def compute(self, keep=False):
        """The timed BC work.  Returns (credited flops, per-product errors
        (depth 0) or None, per-product (x0, y0, C) when keep)."""
        import numpy as np

        if self.impl == "reference":
            R = self.R
            expand = lambda x, u: R.engine._expand(x, u[:, :1], self.mode)  # noqa: E731
            apply = lambda lv, x, y: R.engine.apply_levels(lv, x, y, self.mode)  # noqa: E731
        else:
            from oracle import engine as oracle

            expand = lambda x, u: oracle.combine(x, u[:, :1])  # noqa: E731
            apply = lambda lv, x, y: oracle.apply_levels(lv, x, y, self.mode)  # noqa: E731
        errs, kept = [], []
        with np.errstate(all="ignore"):
            for levels in self.levels:
                x = self.A[None, None]
                y = self.B[None, None]
                for q in range(self.depth):  # branch 0 only: child r = 0 of each level
                    u, v, _ = levels[q]
                    x = expand(x, u)
                    y = expand(y, v)
                try:
                    C = apply(levels[self.depth:], x[:, 0], y[:, 0])
                    errs.append(C)
                except OverflowError:
                    C = None
                    errs.append(None)
                if keep:
                    kept.append((x[:, 0], y[:, 0], C, levels[self.depth:]))
        flops = 2.0 * self.cfg.N ** 3 * len(self.js) / float(self.cfg.rank) ** self.depth
        return flops, errs, kept

    def errors(self, outs):
        """Relative errors (binary64) of the depth-0 products against the
        truth, the reference's own formula when impl is 'reference'
        (experiments.py:258-261); NaN for an overflowed product."""
        import numpy as np

        if self.ref is None:
            return None
        res = []
        for C in outs:
            if C is None:
                res.append(float("nan"))
            elif self.impl == "reference":
                E = self.R.experiments
                res.append(float(E._rel_errors(C, self.ref, E._frob(self.ref), self.mode)[0]))
            else:
                from oracle import engine as oracle

                res.append(float(oracle.rel_errors(C, self.ref)[0]))
        return np.array(res)


def _kind_index(R, kind):
    base = {"uniform_pm1": "uniform", "quadrant100": "gaussian"}.get(kind, kind)
    return R.matgen.MATRIX_KINDS.index(base)


def _ref_generate(R, kind, N, mseed):
    """Operands on the reference's substreams: the reference's own generator
    for its families; the two builder families (BASELINE configs 2 and 4) as
    numpy draws on the same substreams."""
    if kind in R.matgen.MATRIX_KINDS:
        return R.matgen.generate(R.matgen.MatrixSpec(kind, N, mseed))
    ga, gb = R.rng.derive_rng(mseed, 0), R.rng.derive_rng(mseed, 1)
    if kind == "uniform_pm1":
        return 2.0 * ga.random((N, N)) - 1.0, 2.0 * gb.random((N, N)) - 1.0
    if kind == "quadrant100":
        A, B = ga.standard_normal((N, N)), gb.standard_normal((N, N))
        h = N // 2
        A[:h, :h] *= 100.0
        B[h:, h:] *= 100.0
        return A, B
    raise ValueError(kind)


def describe_sample(cfg, count, per_pair, depth, seconds, cores, impl):
    what = f"{count} pair(s) x {per_pair} product(s)"
    if depth:
        what += (f", each product evaluated on branch 0 of its top {depth} level(s) "
                 f"(1/{cfg.rank}^{depth} of the work, credited as 2n^3/{cfg.rank}^{depth}; "
                 "extrapolated)")
    src = ("the unmodified reference randbc (baseline/_ref: _engine.apply_levels on the tables "
           "of randomize._plan_levels / multiply.mode_tensors, as recursive_randomized_apply / "
           "recursive_apply call it)" if impl == "reference"
           else "oracle/engine.py (numpy restatement of randbc._engine)")
    return (f"{what} through {src}, {cores} process(es), {seconds:.1f} s of BC work "
            "(input generation, plan hatting and the binary64 truth untimed)")


def _ref_worker(wid, cfg_name, js, depth, impl, first, steps, barrier, q):
    """Persistent reference-arm worker: prepares its pair once (input
    generation is not the measured path and costs seconds at n=8192), then per
    step waits for all workers, times its BC work, and waits again."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    try:
        job = CpuJob(cfg_name, first + wid, js, depth, impl).prepare()
        for s in range(steps):
            barrier.wait()
            t0 = time.perf_counter()
            flops, _, _ = job.compute()
            t1 = time.perf_counter()
            q.put((s, wid, t0, t1, flops))
            barrier.wait()
    except Exception as exc:  # noqa: BLE001
        q.put(("error", wid, repr(exc), 0, 0))
        barrier.abort()


# per config: reference-arm products per job and subtree depth (each job a
# bounded sample so that --steps 20 --warmup 5 ends within a few minutes)
REF_ARM = {"c1": ((1,), 0), "c2": ((1,), 0), "c3": ((1,), 0), "c4": ((1,), 2), "c5": ((1,), 3)}


def run_reference(args):
    """--impl reference: the reference's own CPU path on all host cores, one
    worker process per core, each step one bounded sample per worker."""
    import multiprocessing as mp

    from paper_1905_07439_b200.configs import get_config

    world, rank, _ = dist_env()
    cfg = get_config(args.config)
    if rank != 0:
        return 0
    impl = cpu_kind()
    cores = os.cpu_count() or 1
    js, depth = REF_ARM[cfg.name]
    steps = args.warmup + args.steps
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(cores)
    q = ctx.Queue()
    procs = [ctx.Process(target=_ref_worker, daemon=True,
                         args=(w, cfg.name, js, depth, impl, 1, steps, barrier, q))
             for w in range(cores)]
    for pr in procs:
        pr.start()
    import queue

    try:
        rows = [q.get(timeout=900) for _ in range(cores * steps)]
    except queue.Empty:
        raise SystemExit("reference arm: a worker stopped reporting") from None
    for pr in procs:
        pr.join(timeout=60)
    bad = [r for r in rows if r[0] == "error"]
    if bad:
        raise SystemExit(f"reference worker failed: {bad[0]}")
    step_s, flops = [], []
    for s in range(args.warmup, steps):
        rs = [r for r in rows if r[0] == s]
        step_s.append(max(r[3] for r in rs) - min(r[2] for r in rs))
        flops.append(sum(r[4] for r in rs))
    total_s = sum(step_s)
    value = sum(flops) / total_s / 1e9
    ms = total_s / args.steps * 1e3
    sample = describe_sample(cfg, cores, len(js), depth, ms / 1e3, cores, impl) + " per step"
    line = {
        "metric": METRIC, "impl": "reference", "value": round(value, 5), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg.mode.label,
        "data": "synthetic (seeded pairs and plans, reference seed layout; no dataset)",
        "config": config_dict(cfg, world, args.trials),
        "cpu_baseline": {"value": round(value, 5), "unit": "GFLOP/s", "cores": cores, "kind": impl,
                         "sample": sample},
        "e2e": {"value": round(value, 5), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(cfg, world, T=None):
    """The `config` object of both arms' lines (identical for one config)."""
    T = T or DEFAULTS[cfg.name]["pairs"]
    return {
        "workload": cfg.name, "desc": cfg.note, "formula": cfg.formula, "Q": cfg.Q, "n": cfg.N,
        "dtype": cfg.mode.label, "pairs_per_rank": T,
        "products_per_pair": cfg.plans_per_pair + 1 if cfg.plans_per_pair > 1 else 2,
        "parallelism": f"trial-sharded x{world}",
        "l2": "operands, binary64 truth and BC intermediates stream through HBM; every level's "
              "working set exceeds the 126 MB L2, so no explicit flush is used",
    }


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
        from paper_1905_07439_b200.configs import packed_plans
        from paper_1905_07439_b200.trials import DeviceErrorTrials

        self.cfg, self.torch = cfg, torch
        self.f = cfg.formula_obj()
        self.A, self.B = A, B
        self.pair_ids = list(pair_ids)
        self.packed = packed_plans(cfg, [cfg.plan_key(p) for p in pair_ids])
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
        self.e2e_single_ms = ms
        # the same calls as a stream (rbc_error_trials_begin / _end, at most two
        # in flight): step s+1 is submitted before step s's result is taken, so
        # its operands are copied while step s computes; every step's H2D and
        # D2H is inside the timed region
        from paper_1905_07439_b200.trials import ErrorTrialStream

        st = ErrorTrialStream(self.f, self.cfg.Q, self.cfg.mode)
        An, Bn = A_pin.numpy(), B_pin.numpy()
        first = st.result(st.submit(An, Bn, packed=pn))
        if not (np.array_equal(first["err_rand"], err_r, equal_nan=True)
                and np.array_equal(first["err_det"], err_d, equal_nan=True)):
            raise SystemExit("streamed e2e errors differ from the device-resident run")
        with no_gc():
            prev = st.submit(An, Bn, packed=pn)  # untimed: fills the pipeline
            t0 = time.perf_counter()
            for _ in range(steps):
                cur = st.submit(An, Bn, packed=pn)
                last = st.result(prev)
                prev = cur
            ms = (time.perf_counter() - t0) / steps * 1e3
            last = st.result(prev)
        if not np.array_equal(last["err_rand"], err_r, equal_nan=True):
            raise SystemExit("streamed e2e errors differ from the device-resident run")
        h2d = self.A.nbytes + self.B.nbytes + self.packed.nbytes
        d2h = 2 * len(err_r) * 9
        return ms, h2d, d2h


    def fresh(self, steps, warmup=2):
        """Fresh inputs every step: the step's operand pairs drawn on the GPU
        (rbc_matgen from keys of the native SeedSequence), its plans drawn on
        the host (native draw_plan) and copied H2D, the error trials run, the
        per-trial errors copied D2H; wall clock per step over a run of steps
        (trials.run_trial_set: the next step's pairs are drawn on a second
        stream while a step computes).  Pairs continue after the resident set
        (no pair is reused)."""
        import torch

        from paper_1905_07439_b200.trials import run_trial_set

        cfg, T = self.cfg, len(self.pair_ids)
        p0 = self.pair_ids[-1] + 1
        dev = self.a.device
        runners = {T: self.runner}
        run_trial_set(cfg, p0, warmup * T, T, dev, True, runners)
        torch.cuda.synchronize()
        with no_gc():
            t0 = time.perf_counter()
            run_trial_set(cfg, p0 + warmup * T, steps * T, T, dev, True, runners)
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) / steps * 1e3
        return ms


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
    feeds the timed region.  The first full-size call also pays the one-time
    allocations (torch's caching allocator growing to the outputs, the
    generator's word and map buffers), which is what made round 1's single
    timing vary (671 vs 35-73 ms); the steady figure is the median of three
    later calls."""
    import torch

    from paper_1905_07439_b200.configs import make_pairs_device

    make_pairs_device(cfg, first, min(T, 2))  # warm-up (module load, small buffers)
    times = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dA, dB = make_pairs_device(cfg, first, T)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        if len(times) < 4:
            del dA, dB
    same = (dA.cpu().numpy().tobytes() == A.tobytes() and dB.cpu().numpy().tobytes() == B.tobytes())
    del dA, dB
    return {"kind": cfg.kind, "device_matgen_first_call_ms": round(times[0] * 1e3, 2),
            "device_matgen_ms": round(statistics.median(times[1:]) * 1e3, 2),
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

        # RBC_BENCH_BACKEND=gloo: test hook (tests/test_multiprocess_gpu.py) --
        # ranks share the visible GPUs and the statistics collectives go over
        # gloo on host tensors; the driver's runs use NCCL, one GPU per rank
        backend = os.environ.get("RBC_BENCH_BACKEND", "nccl")
        torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group(backend)
    else:
        dist = None
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    coll = None if (dist is not None and dist.get_backend() == "gloo") else dev  # collective tensors
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

    tmax = distributed.max_over_ranks([dev_ms, e2e[0] if e2e else 0.0], device=coll)
    dev_ms = float(tmax[0])
    allerr = distributed.gather_trials(
        np.stack([err_r, nf_r.astype(np.float64)]), device=coll)
    alldet = distributed.gather_trials(np.stack([err_d, nf_d.astype(np.float64)]), device=coll)
    if args.dump_errors and rank == 0:  # per-trial errors of all ranks, trial order
        np.savez(args.dump_errors, err_rand=allerr[0], nf_rand=allerr[1], err_det=alldet[0],
                 nf_det=alldet[1])

    flops_step = 2.0 * cfg.N ** 3 * wl.products * world
    value = flops_step / (dev_ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dev_ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg.mode.label,
        "data": "synthetic (seeded pairs and plans, reference seed layout; no dataset)",
        "trials_per_s": round(T * world / (dev_ms / 1e3), 3),
        "products_per_s": round(wl.products * world / (dev_ms / 1e3), 3),
        "config": config_dict(cfg, world, args.trials),
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
    if hasattr(wl, "fresh") and not args.no_e2e:
        # the host-buffer calls above keep an arena sized to most of the free
        # memory; give it back before the device-resident runner allocates
        from paper_1905_07439_b200 import _lib as _rbclib
        _rbclib.check(_rbclib.load().rbc_release_device_memory())
        barrier()
        fresh_ms = float(distributed.max_over_ranks([wl.fresh(args.steps)], device=coll)[0])
        line["e2e_fresh_inputs"] = {
            "value": round(flops_step / (fresh_ms / 1e3) / 1e9, 3), "unit": "GFLOP/s",
            "ms_per_step": round(fresh_ms, 3),
            "what": "every step draws new operand pairs on the GPU (rbc_matgen; keys from the "
                    "native SeedSequence), new plans on the host (native draw_plan, copied H2D), "
                    "runs the error trials and copies the errors D2H; wall clock",
            "ratio_to_resident_step": round(fresh_ms / dev_ms, 3),
        }
    if e2e is not None:
        e2e_ms = float(tmax[1])
        line["e2e"] = {"value": round(flops_step / (e2e_ms / 1e3) / 1e9, 3), "unit": "GFLOP/s",
                       "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": int(e2e[1]),
                       "d2h_bytes_per_step": int(e2e[2]),
                       "path": "public host-buffer call (error_trials / average_trials, C ABI "
                               "rbc_error_trials): pinned host operands and plans copied H2D, "
                               "per-trial errors copied D2H, inside the timed region"}
        single = getattr(wl, "e2e_single_ms", None)
        if single is not None:
            line["e2e"]["path"] = (
                "public host-buffer calls as a stream (trials.ErrorTrialStream, C ABI "
                "rbc_error_trials_begin / _end, two calls in flight): every step's pinned host "
                "operands and plans copied H2D and its per-trial errors copied D2H inside the timed "
                "region; step s+1's copies overlap step s's kernels")
            single = float(distributed.max_over_ranks([single], device=coll)[0])
            line["e2e"]["single_call"] = {
                "ms_per_step": round(single, 3),
                "value": round(flops_step / (single / 1e3) / 1e9, 3), "unit": "GFLOP/s",
                "what": "one synchronous rbc_error_trials call per step (begin + end back to "
                        "back): the GPU idles during each call's first copy"}
            calls = getattr(wl, "e2e_calls", None)
            if calls:
                line["e2e"]["single_call"]["ms_per_call"] = [round(c, 2) for c in calls]
    del wl
    torch.cuda.empty_cache()

    if not args.no_tts and cfg.plans_per_pair > 1:
        barrier()
        line["time_to_solution"] = time_to_solution_average(cfg, T, dev, rank, world, coll)
    if not args.no_tts and cfg.plans_per_pair == 1:
        barrier()
        line["time_to_solution"] = time_to_solution(cfg, T, dev, rank, world, coll)
        tts_err = line["time_to_solution"].pop("_errors")
        if args.dump_errors and rank == 0:
            np.savez(args.dump_errors + ".tts.npz", err_rand=tts_err[0], err_det=tts_err[1])
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_leg(cfg, first, T, err_r, err_d)
        line["cpu_baseline"] = cpu
        tts = line.get("time_to_solution")
        if tts:
            per_product_s = cpu.pop("_seconds_per_product")
            tts["cpu_1core_extrapolated_s"] = round(per_product_s * 2 * cfg.trials, 1)
            tts["cpu_note"] = ("the cpu_baseline sample's seconds per full product x 2 products x "
                               f"{cfg.trials} pairs, one process; BC products only (input "
                               "generation and the binary64 truth excluded)")
            tts["speedup_vs_cpu_1core"] = round(tts["cpu_1core_extrapolated_s"] / tts["seconds"], 1)
        else:
            cpu.pop("_seconds_per_product", None)
    if rank == 0 and world == 1 and not args.no_dropin:
        line["dropin_e2e"] = dropin_e2e()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def cpu_baseline_leg(cfg, first, T, err_r, err_d):
    """The reference's CPU path on one core over a bounded sample of the
    workload (rank 0, N=1), and the parity of the GPU run against it: the
    per-trial errors of whole products (configs 1-3), or, where one CPU
    product takes minutes (configs 4-5), the branch-0 sub-products bit for bit
    against the GPU engine run on the same sub-operands through the drop-in
    (reference _engine.apply_levels signature)."""
    import numpy as np

    from paper_1905_07439_b200 import engine

    count, per_pair, depth = DEFAULTS[cfg.name]["cpu"]
    count = min(count, T)
    impl = cpu_kind()
    js = tuple(range(per_pair)) if cfg.plans_per_pair > 1 else ((0, 1) if per_pair == 2 else (1,))
    total_s, flops, agree, branch = 0.0, 0.0, [], []
    for i, p in enumerate(range(first, first + count)):
        job = CpuJob(cfg.name, p, js, depth, impl).prepare()
        t0 = time.perf_counter()
        fl, outs, kept = job.compute(keep=depth > 0)
        total_s += time.perf_counter() - t0
        flops += fl
        if depth == 0:
            want = job.errors(outs)
            G = cfg.plans_per_pair
            got = np.array([err_d[i] if j == 0 else (err_r[i * G + j - 1] if G > 1 else err_r[i])
                            for j in js])
            agree.append(bool(np.allclose(got, want, rtol=1e-12, atol=0, equal_nan=True)))
        else:
            for x0, y0, C, lv in kept:
                try:
                    Cg = engine.apply_levels(lv, x0, y0, job.mode)
                except OverflowError:
                    Cg = None
                branch.append((C is None and Cg is None) or
                              (C is not None and Cg is not None and np.array_equal(C, Cg)))
        del job
    out = {
        "value": round(flops / total_s / 1e9, 6), "unit": "GFLOP/s", "cores": 1, "kind": impl,
        "sample": describe_sample(cfg, count, len(js), depth, total_s, 1, impl),
        "errors_agree_with_gpu": all(agree) if agree else None,
        "_seconds_per_product": total_s / (count * len(js)) * float(cfg.rank) ** depth,
    }
    if depth == 0:
        out["errors_compared"] = f"{count} pair(s) x {len(js)} product(s), rtol 1e-12"
    else:
        out["branch_products_bitwise_equal"] = all(branch)
        out["branch_products_compared"] = (
            f"{len(branch)} branch-0 sub-product(s) at n={cfg.N // cfg.n ** depth} "
            f"(levels {depth}..{cfg.Q - 1}), CPU vs GPU engine (engine.apply_levels), "
            "values and overflow")
        out["errors_agree_with_gpu"] = all(branch)
    return out


def time_to_solution(cfg, T_step, dev, rank, world, coll=None):
    """Wall-clock time for the config's whole trial set (e.g. configuration 5:
    all 64 pairs), strong-scaled over the ranks: each rank draws its share of
    the pairs on the GPU (rbc_matgen, bit-identical to the host draw), runs
    the error trials T_step pairs at a time and copies the errors back; the
    figure is the max over ranks."""
    import numpy as np
    import torch

    from paper_1905_07439_b200 import distributed

    total = cfg.trials
    per = -(-total // world)
    lo, hi = 1 + rank * per, min(total, (rank + 1) * per)
    runners = {}
    from paper_1905_07439_b200.trials import run_trial_set

    def whole(pipelined):
        run_trial_set(cfg, lo, min(T_step, hi - lo + 1), T_step, dev, pipelined, runners)  # warm-up
        torch.cuda.synchronize()
        distributed.barrier_if(world)
        t0 = time.perf_counter()
        er, ed, _, _ = run_trial_set(cfg, lo, hi - lo + 1, T_step, dev, pipelined, runners)
        sec = time.perf_counter() - t0
        return float(distributed.max_over_ranks([sec], device=coll)[0]), np.stack([er, ed])

    serial_sec, e_serial = whole(False)
    sec, e = whole(True)
    same = bool(np.array_equal(e, e_serial, equal_nan=True))
    if total % world == 0:  # equal shards: gather in rank (= pair) order
        e = distributed.gather_trials(e, device=coll)
    return {
        "pairs": total, "products": 2 * total, "seconds": round(sec, 3), "scaling": "strong",
        "n_gpus": world, "pairs_per_launch": T_step,
        "what": "wall clock, all pairs: device input generation, plans, binary64 truth, "
                "deterministic + randomized products, errors copied to the host (max over ranks); "
                "the next pass's inputs are drawn on a second stream while a pass computes "
                "(trials.run_trial_set)",
        "seconds_unpipelined": round(serial_sec, 3), "pipelined_equals_unpipelined": same,
        # None when every trial overflowed (config 4's deterministic products)
        "err_rand_mean": float(np.nanmean(e[0])) if np.isfinite(e[0]).any() else None,
        "err_det_mean": float(np.nanmean(e[1])) if np.isfinite(e[1]).any() else None,
        "_errors": e,
    }


def time_to_solution_average(cfg, P_step, dev, rank, world, coll=None):
    """Wall-clock time for an averaging config's whole trial set (configuration
    3: 500 pairs x 32 plans), strong-scaled over the ranks: pairs drawn on the
    GPU, plans drawn natively and hatted on the host, the averaging pipeline
    P_step pairs at a time (trials.run_average_set); max over ranks."""
    import numpy as np
    import torch

    from paper_1905_07439_b200 import distributed
    from paper_1905_07439_b200.trials import run_average_set

    total = cfg.trials
    per = -(-total // world)
    lo, hi = 1 + rank * per, min(total, (rank + 1) * per)

    def whole(pipelined):
        run_average_set(cfg, lo, min(2 * P_step, hi - lo + 1), P_step, dev, pipelined)  # warm-up
        torch.cuda.synchronize()
        distributed.barrier_if(world)
        t0 = time.perf_counter()
        r = run_average_set(cfg, lo, hi - lo + 1, P_step, dev, pipelined)
        sec = time.perf_counter() - t0
        return float(distributed.max_over_ranks([sec], device=coll)[0]), r

    serial_sec, rs = whole(False)
    sec, r = whole(True)
    same = all(r[k].tobytes() == rs[k].tobytes() for k in ("err_rand", "err_mean", "err_det"))
    G = cfg.plans_per_pair
    return {
        "pairs": total, "products": (G + 1) * total, "seconds": round(sec, 3), "scaling": "strong",
        "n_gpus": world, "pairs_per_launch": P_step,
        "what": "wall clock, all pairs of this rank's share: device input generation, native plan "
                "draws, host hatting of the dense tables, binary64 truth, deterministic + G "
                "randomized products, per-plan and running-mean errors copied to the host (max "
                "over ranks); the next pass is prepared while a pass computes "
                "(trials.run_average_set)",
        "seconds_unpipelined": round(serial_sec, 3), "pipelined_equals_unpipelined": same,
        "err_rand_mean": float(np.nanmean(r["err_rand"])), "err_det_mean": float(np.nanmean(r["err_det"])),
        "err_mean_at_G": float(np.nanmean(r["err_mean"][:, -1])),
    }


def dropin_e2e():
    """The reference's own workflow through the drop-in: the shipped command
    `randbc experiment s2-variants --seed 1` (n=320, Q=1..5, 100 plans, all six
    input families, f32; reference README.md:108-109 "around ten minutes",
    test_acceptance.py:330-365 caps it at 1800 s) run by the unmodified
    reference (baseline/_ref) with engine.install(), wall clock; its CSV is
    compared with the reference's artifact (tests/golden/s2_variants_320.csv,
    rel_error to 1e-12)."""
    import io

    import numpy as np

    if not reference_available():
        return {"unavailable": "baseline/_ref (the unmodified reference) is not installed"}
    from paper_1905_07439_b200 import engine

    R = reference_modules()
    import randbc.cli

    want = (ROOT / "tests" / "golden" / "s2_variants_320.csv").read_text().splitlines()

    def table(lines):
        hdr = lines[0].split(",")
        k = hdr.index("rel_error")
        return {tuple(x for i, x in enumerate(row.split(",")) if i != k): float(row.split(",")[k])
                for row in lines[1:]}

    tw = table(want)

    def run(wide):
        engine.install(R.engine, wide=wide)
        try:
            with tempfile.TemporaryDirectory() as d:
                out = Path(d) / "s2.csv"
                sink = io.StringIO()
                t0 = time.perf_counter()
                with contextlib.redirect_stdout(sink):
                    code = randbc.cli.main(["experiment", "s2-variants", "--seed", "1", "--out", str(out)])
                sec = time.perf_counter() - t0
                got = out.read_text().splitlines() if code == 0 else []
        finally:
            engine.uninstall(R.engine)
        tg = table(got) if got else {}
        match = bool(got) and tg.keys() == tw.keys() and all(
            np.isclose(tg[key], tw[key], rtol=1e-12, atol=0) for key in tw)
        return sec, code, len(got) - 1 if got else 0, match

    sec, code, rows, match = run(False)  # the device is warm: the bench steps ran before
    wsec, wcode, wrows, wmatch = run(True)
    return {
        "workload": "randbc experiment s2-variants --seed 1 (reference CLI defaults: n=320, "
                    "Q=1..5, 100 plans, 6 input families, f32) with engine.install()",
        "seconds": round(sec, 2), "exit_code": code, "rows": rows,
        "matches_reference_artifact": match,
        "wide": {"seconds": round(wsec, 2), "exit_code": wcode, "rows": wrows,
                 "matches_reference_artifact": wmatch,
                 "what": "engine.install(wide=True): the reference's L2 entry points and "
                         "experiments._rel_errors routed to this package as well (plans instead "
                         "of hatted tables, device-side scalings and error reductions)"},
        "reference_published": "around ten minutes (README.md:108-109); acceptance cap 1800 s "
                               "(tests/test_acceptance.py:365)",
    }


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
