"""GPU: bench.py's multi-rank path (torchrun, trial sharding, max-over-ranks
timing, gathered per-trial errors, the strong-scaled time-to-solution run)
with two processes on librbc.so, against the single-process run bit for bit.

Both ranks share the one visible B200 (RBC_BENCH_BACKEND=gloo: the statistics
collectives go over gloo on host tensors); the driver's scaling runs use one
GPU per rank and NCCL, with the same sharding and gather code."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(tmp, world, per_rank, tag):
    dump = str(tmp / f"{tag}.npz")
    args = ["--config", "c1", "--steps", "2", "--warmup", "3", "--trials", str(per_rank),
            "--no-cpu", "--no-e2e", "--no-dropin", "--dump-errors", dump, "--gpus", str(world)]
    env = dict(os.environ, RBC_BENCH_BACKEND="gloo", PYTHONPATH=str(ROOT))
    if world == 1:
        cmd = [sys.executable, str(ROOT / "bench.py"), *args]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
               str(_free_port()), str(ROOT / "bench.py"), *args]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    line = json.loads([x for x in res.stdout.splitlines() if x.startswith("{")][-1])
    return line, np.load(dump), np.load(dump + ".tts.npz")


def test_two_ranks_equal_single_process(tmp_path):
    from paper_1905_07439_b200 import _lib

    _lib.require_device()
    two, e2, t2 = _run(tmp_path, 2, 50, "two")   # pairs 1-50 on rank 0, 51-100 on rank 1
    one, e1, t1 = _run(tmp_path, 1, 100, "one")  # pairs 1-100 in one process
    assert two["n_gpus"] == 2 and one["n_gpus"] == 1
    for k in ("err_rand", "nf_rand", "err_det", "nf_det"):
        assert e1[k].shape == (100,) and np.array_equal(e1[k], e2[k], equal_nan=True), k
    assert two["errors"] == one["errors"]
    # strong-scaled time to solution: all 100 pairs of configuration 1 split
    # over the ranks; the gathered errors equal the one-process run's
    assert two["time_to_solution"]["pairs"] == one["time_to_solution"]["pairs"] == 100
    assert np.array_equal(t1["err_rand"], t2["err_rand"])
    assert np.array_equal(t1["err_det"], t2["err_det"])
    assert np.array_equal(t1["err_rand"], e1["err_rand"])
