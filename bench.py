#!/usr/bin/env python
"""Benchmark of the randomized BC multiply hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A *step* is one pass of the hot path over one batch of synthetic input: for
each of the rank's T operand pairs (config's seed layout) the
binary64 truth, the deterministic BC product and its error, and the
randomized BC product (fresh per-level signed permutations) and its error.
Default workload: BASELINE.json configs[1] ("c2": Laderman <3,3,3;23>,
Q=4, n=243, f32, Uniform[-1,1], 1000 pairs per rank).

value  : effective GFLOP/s = 2 n^3 x (2 BC products per pair) x T x ranks
         / step time, inputs resident in HBM, CUDA events on the launch
         stream, max over ranks
e2e    : the same through the public host-buffer C-ABI call
         (rbc_error_trials): pinned host operands + plans copied H2D and
         per-trial errors copied D2H inside the timed region
roofline: the stage with the largest share of the timed region, from the
         engine's CUDA-event stage profiler (algorithmic bytes or flops per
         launch / average launch duration) against MEASURED_PEAKS.json
cpu_baseline: the CPU oracle (numpy restatement of the reference engine,
         oracle/) on a bounded sample of the same pairs, rank 0, 1 core
--impl reference: the CPU oracle arm with all host cores (the reference is
         pure Python/numpy and cannot be compiled into oracle/_ref)

Multi-GPU: one process per GPU (torchrun), each rank takes its own block of
pairs (weak scaling); the only collective is the MAX of the step times and
an all-gather of the per-trial error statistics (tiny, NCCL).
"""

from __future__ import annotations

import argparse
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--trials", type=int, default=0, help="pairs per rank (default: config)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=0, help="pairs in the CPU baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


# --------------------------------------------------------------- helpers ----
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


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
        return d.get("hbm_gbs", HBM_FALLBACK_GBS), "measured"
    return HBM_FALLBACK_GBS, "fallback"


def fp_peaks():
    """Exact-order (FMUL+FADD) CUDA-core peaks measured by tools/fp_peak.py."""
    p = ROOT / "profiles" / "fp_peaks.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured (profiles/fp_peaks.json)"
    return {"f32_tflops": FP32_NOMINAL_TFLOPS, "f64_tflops": FP32_NOMINAL_TFLOPS / 2,
            "f16_tflops": FP32_NOMINAL_TFLOPS * 2}, "nominal"


def ncu_traffic(stage: str, config: str):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(config, {}).get(stage)


def roofline(prof: dict, config: str):
    if not prof:
        return None
    stage, agg = max(prof.items(), key=lambda kv: kv[1]["ms"])
    avg_s = agg["ms"] / agg["count"] / 1e3
    per_launch_bytes = agg["bytes"] / agg["count"]
    per_launch_flops = agg["flops"] / agg["count"]
    total_ms = sum(v["ms"] for v in prof.values())
    if stage.startswith(("leaf", "truth")):
        peaks, how = fp_peaks()
        key = {"leaf_f32": "f32_tflops", "leaf_f16": "f16_tflops"}.get(stage, "f64_tflops")
        achieved = per_launch_flops / avg_s / 1e12
        peak = peaks[key]
        bound, unit = ("cuda-core-" + key.split("_")[0]), "TFLOP/s"
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
def _cpu_pair_work(args):
    """One pair through the CPU oracle: truth, deterministic and randomized
    products, both errors (the same step definition as the GPU arm)."""
    cfg_name, p = args
    import numpy as np

    from oracle import engine as oracle
    from paper_1905_07439_b200.configs import get_config
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.randomize import plan_levels

    cfg = get_config(cfg_name)
    f = cfg.formula_obj()
    A, B = cfg.pair(p)
    ref = oracle.standard_multiply(A.astype(np.float64), B.astype(np.float64))
    det_levels = [mode_tensors(f, cfg.mode)] * cfg.Q
    rp = cfg.plan(cfg.plan_key(p))
    rand_levels = [plan_levels(f, [rp.levels[q]], cfg.mode) for q in range(cfg.Q)]
    out = []
    with np.errstate(all="ignore"):
        for levels in (det_levels, rand_levels):
            try:
                C = oracle.apply_levels(levels, A[None], B[None], cfg.mode)
                out.append(float(oracle.rel_errors(C, ref)[0]))
            except OverflowError:
                out.append(float("nan"))
    return out


def cpu_oracle_rate(cfg, pairs, workers: int):
    import concurrent.futures as cf

    jobs = [(cfg.name, p) for p in pairs]
    t0 = time.perf_counter()
    if workers > 1:
        with cf.ProcessPoolExecutor(max_workers=workers) as ex:
            res = list(ex.map(_cpu_pair_work, jobs))
    else:
        res = [_cpu_pair_work(j) for j in jobs]
    dt = time.perf_counter() - t0
    return dt, res


def default_cpu_sample(cfg) -> int:
    # about 10-30 s of single-core oracle work
    return {"c1": 40, "c2": 8, "c3": 1, "c4": 1, "c5": 1}.get(cfg.name, 2)


# ------------------------------------------------------------ reference ----
def run_reference(args):
    from paper_1905_07439_b200.configs import get_config

    world, rank, _ = dist_env()
    cfg = get_config(args.config)
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    per_step = max(cores, 1)
    flops_per_pair = 2 * cfg.effective_flops()
    p = 1
    for _ in range(args.warmup):
        cpu_oracle_rate(cfg, range(p, p + per_step), cores)
        p += per_step
    total = 0.0
    for _ in range(args.steps):
        dt, _ = cpu_oracle_rate(cfg, range(p, p + per_step), cores)
        total += dt
        p += per_step
    ms = total / args.steps * 1e3
    value = flops_per_pair * per_step / (ms / 1e3) / 1e9
    line = {
        "metric": "effective GFLOP/s (2n^3/time) of randomized BC matmul error trials",
        "impl": "reference", "value": round(value, 4), "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg.mode.label,
        "data": "synthetic (seeded, reference seed layout)",
        "trials_per_s": round(per_step / (ms / 1e3), 4),
        "config": {"workload": cfg.name, "desc": cfg.note, "pairs_per_step": per_step},
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"{per_step} pairs per step through oracle/engine.py "
                                   f"(numpy restatement of randbc._engine), one process per core"},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ ours ----
def run_ours(args):
    import numpy as np
    import torch

    from paper_1905_07439_b200 import _lib
    from paper_1905_07439_b200.configs import get_config, make_pairs
    from paper_1905_07439_b200.randomize import pack_recursive_plans
    from paper_1905_07439_b200.trials import DeviceErrorTrials, error_trials

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

    from paper_1905_07439_b200 import distributed

    cfg = get_config(args.config)
    T = args.trials or cfg.trials
    f = cfg.formula_obj()
    first, _ = distributed.shard(rank, world, T)
    pair_ids = distributed.pair_ids(rank, world, T)
    workers = min(32, max(1, (os.cpu_count() or 2) // max(1, world)))
    A, B = make_pairs(cfg, first, T, workers=workers)
    packed = pack_recursive_plans([cfg.plan(cfg.plan_key(p)) for p in pair_ids], cfg.Q, cfg.n)

    a_d = torch.from_numpy(A).to(dev)
    b_d = torch.from_numpy(B).to(dev)
    pl_d = torch.from_numpy(packed).to(dev)
    runner = DeviceErrorTrials(f, cfg.Q, cfg.N, cfg.mode, T, device=dev)
    stream = torch.cuda.Stream(device=dev)

    def barrier():
        if dist is not None:
            dist.barrier()

    clocks = Clocks(local)
    clocks.start()
    for _ in range(args.warmup):
        runner.run(a_d, b_d, pl_d, stream=stream)
    torch.cuda.synchronize()
    barrier()
    _lib.profile_enable(True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        runner.run(a_d, b_d, pl_d, stream=stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    prof = _lib.profile_summary()
    _lib.profile_enable(False)
    launches = sum(v["count"] for v in prof.values())
    dev_ms = ev0.elapsed_time(ev1) / args.steps

    err_r = runner.err_rand.cpu().numpy()
    err_d = runner.err_det.cpu().numpy()
    nf_r = runner.nf_rand.cpu().numpy().astype(bool)
    nf_d = runner.nf_det.cpu().numpy().astype(bool)

    # ---- e2e through the public host-buffer call
    e2e_ms = None
    h2d = A.nbytes + B.nbytes + packed.nbytes
    d2h = 2 * T * 8 + 2 * T
    if not args.no_e2e:
        A_pin = torch.from_numpy(A).pin_memory().numpy()
        B_pin = torch.from_numpy(B).pin_memory().numpy()
        P_pin = torch.from_numpy(packed).pin_memory().numpy()
        res = error_trials(f, cfg.Q, A_pin, B_pin, cfg.mode, packed=P_pin)
        same = (np.array_equal(res["err_rand"], err_r, equal_nan=True)
                and np.array_equal(res["err_det"], err_d, equal_nan=True))
        if not same:
            raise SystemExit("e2e errors differ from the device-resident run")
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            error_trials(f, cfg.Q, A_pin, B_pin, cfg.mode, packed=P_pin)
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) / args.steps * 1e3

    # ---- max over ranks + gather of per-trial statistics
    tmax = distributed.max_over_ranks([dev_ms, e2e_ms or 0.0], device=dev)
    dev_ms, e2e_ms = float(tmax[0]), (float(tmax[1]) if e2e_ms is not None else None)
    allerr = distributed.gather_trials(
        np.stack([err_r, err_d, nf_r.astype(np.float64), nf_d.astype(np.float64)]), device=dev)
    err_r_all, err_d_all = allerr[0], allerr[1]
    nf_r_all, nf_d_all = allerr[2] > 0, allerr[3] > 0

    flops_step = 2 * cfg.effective_flops() * T * world
    value = flops_step / (dev_ms / 1e3) / 1e9
    line = {
        "metric": "effective GFLOP/s (2n^3/time) of randomized BC matmul error trials",
        "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dev_ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": cfg.mode.label,
        "data": "synthetic (seeded pairs and plans, reference seed layout; no dataset)",
        "trials_per_s": round(T * world / (dev_ms / 1e3), 2),
        "config": {
            "workload": cfg.name, "desc": cfg.note, "formula": cfg.formula, "Q": cfg.Q,
            "n": cfg.N, "pairs_per_rank": T, "products_per_pair": 2,
            "parallelism": f"trial-sharded x{world}",
            "l2": f"inputs {A.nbytes * 2 / 1e6:.0f} MB + truth {T * cfg.N ** 2 * 8 / 1e6:.0f} MB "
                  "per step exceed the 126 MB L2 (no flush needed)",
        },
        "gpu_launches": launches,
        "clocks": clk,
        "roofline": roofline(prof, cfg.name),
        "errors": distributed.trial_stats(err_r_all, err_d_all, nf_r_all, nf_d_all),
    }
    if e2e_ms is not None:
        line["e2e"] = {"value": round(flops_step / (e2e_ms / 1e3) / 1e9, 3), "unit": "GFLOP/s",
                       "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": int(h2d),
                       "d2h_bytes_per_step": int(d2h)}

    # ---- CPU baseline (rank 0, N = 1)
    if rank == 0 and world == 1 and not args.no_cpu:
        S = args.cpu_sample or default_cpu_sample(cfg)
        dt, res = cpu_oracle_rate(cfg, pair_ids[:S], 1)
        cpu_val = 2 * cfg.effective_flops() * S / dt / 1e9
        got = np.stack([err_d[:S], err_r[:S]], axis=1)
        want = np.array(res)
        agree = bool(np.allclose(got, want, rtol=1e-10, atol=0, equal_nan=True))
        line["cpu_baseline"] = {
            "value": round(cpu_val, 5), "unit": "GFLOP/s", "cores": 1, "kind": "port",
            "sample": f"first {S} pairs of the step through oracle/engine.py (numpy restatement "
                      f"of randbc._engine), {dt:.1f} s", "errors_agree_with_gpu": agree,
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
