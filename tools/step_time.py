"""Time the error-trial step without the stage profiler (concurrent lanes on).
    python tools/step_time.py <config> [pairs] [steps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1905_07439_b200.configs import get_config, make_pairs  # noqa: E402

cfg = get_config(sys.argv[1])
T = int(sys.argv[2]) if len(sys.argv) > 2 else bench.DEFAULTS[cfg.name]["pairs"]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
A, B = make_pairs(cfg, 1, T, workers=16)
kind = bench.AverageWorkload if cfg.plans_per_pair > 1 else bench.ErrorTrialWorkload
wl = kind(cfg, list(range(1, T + 1)), A, B, torch.device("cuda:0"), torch)
st = torch.cuda.Stream()
for _ in range(3):
    wl.run(st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(steps):
    wl.run(st)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"{cfg.name} T={T} {ms:.3f} ms/step  {2.0 * cfg.N ** 3 * wl.products / (ms / 1e3) / 1e9:.1f} GFLOP/s")
