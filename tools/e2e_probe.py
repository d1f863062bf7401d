"""Probe the host-buffer (e2e) path: H2D bandwidth and per-call times."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_07439_b200.configs import get_config, make_pairs  # noqa: E402
from paper_1905_07439_b200.randomize import pack_recursive_plans  # noqa: E402
from paper_1905_07439_b200.trials import error_trials  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
T = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.trials
A, B = make_pairs(cfg, 1, T, workers=16)
packed = pack_recursive_plans([cfg.plan(p) for p in range(1, T + 1)], cfg.Q, cfg.n)
Ap = torch.from_numpy(A).pin_memory()
Bp = torch.from_numpy(B).pin_memory()
Pp = torch.from_numpy(packed).pin_memory()
print("pinned:", Ap.is_pinned(), Bp.is_pinned())
d = torch.empty_like(Ap, device="cuda")
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d.copy_(Ap, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"H2D {Ap.numel() * Ap.element_size() / 1e6:.0f} MB in {dt * 1e3:.2f} ms = {Ap.numel() * Ap.element_size() / dt / 1e9:.1f} GB/s")
An, Bn, Pn = Ap.numpy(), Bp.numpy(), Pp.numpy()
times = []
f = cfg.formula_obj()
for i in range(int(sys.argv[3]) if len(sys.argv) > 3 else 12):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    error_trials(f, cfg.Q, An, Bn, cfg.mode, packed=Pn)
    torch.cuda.synchronize()
    times.append((time.perf_counter() - t0) * 1e3)
import statistics  # noqa: E402
print("calls ms:", " ".join(f"{t:.1f}" for t in times))
print(f"median {statistics.median(times[2:]):.2f} ms  min {min(times[2:]):.2f} ms")
