"""Wall clock of trials.run_trial_set against the number of passes (GPU box):
    python tools/experiments/trial_set_probe.py [config] [pairs per pass]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

from paper_1905_07439_b200.configs import get_config  # noqa: E402
from paper_1905_07439_b200.trials import run_trial_set  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "c4")
T = int(sys.argv[2]) if len(sys.argv) > 2 else 16
runners = {}
run_trial_set(cfg, 1, 2 * T, T, "cuda:0", True, runners)
for pipelined in (True, False):
    for steps in (1, 2, 4, 8, 16):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run_trial_set(cfg, 1, steps * T, T, "cuda:0", pipelined, runners)
        ms = (time.perf_counter() - t0) * 1e3
        print(f"{cfg.name} pipelined={pipelined} passes={steps:2d} total {ms:8.2f} ms  per pass {ms / steps:7.2f}", flush=True)
