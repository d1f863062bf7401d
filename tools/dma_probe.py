"""H2D copy rate with and without the c2 step running beside it (GPU box):
is the host-buffer pipeline's copy stream slowed by the kernels' HBM traffic?
    python tools/dma_probe.py [config]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1905_07439_b200.configs import get_config, make_pairs  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
T = bench.DEFAULTS[cfg.name]["pairs"]
A, B = make_pairs(cfg, 1, T, workers=16)
dev = torch.device("cuda", 0)
wl = bench.ErrorTrialWorkload(cfg, list(range(1, T + 1)), A, B, dev, torch)
s_comp = torch.cuda.Stream()
s_copy = torch.cuda.Stream()
host = torch.from_numpy(A).pin_memory()
dst = torch.empty_like(host, device=dev)
nbytes = host.numel() * host.element_size()
for _ in range(3):
    wl.run(s_comp)
torch.cuda.synchronize()


def timed_copy():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s_copy):
        e0.record(s_copy)
        dst.copy_(host, non_blocking=True)
        e1.record(s_copy)
    return e0, e1


for label, busy in (("idle", False), ("beside the c2 step", True), ("idle", False)):
    rates = []
    for _ in range(3):
        torch.cuda.synchronize()
        if busy:
            wl.run(s_comp)
            wl.run(s_comp)
        e0, e1 = timed_copy()
        torch.cuda.synchronize()
        rates.append(nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    print(f"H2D {nbytes / 1e6:.0f} MB {label}: " + " ".join(f"{r:.1f}" for r in rates) + " GB/s")

# the pipeline's pattern: A and B of each of 16 chunks, back to back on one stream
hostB = torch.from_numpy(B).pin_memory()
dstB = torch.empty_like(hostB, device=dev)
nch = 16
step = (T + nch - 1) // nch


def chunked():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s_copy):
        e0.record(s_copy)
        for c in range(0, T, step):
            dst[c:c + step].copy_(host[c:c + step], non_blocking=True)
            dstB[c:c + step].copy_(hostB[c:c + step], non_blocking=True)
        e1.record(s_copy)
    return e0, e1


for label, busy in (("idle", False), ("beside the c2 step", True)):
    rates = []
    for _ in range(3):
        torch.cuda.synchronize()
        if busy:
            wl.run(s_comp)
            wl.run(s_comp)
        e0, e1 = chunked()
        torch.cuda.synchronize()
        rates.append(2 * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    print(f"H2D {2 * nbytes / 1e6:.0f} MB in {2 * nch} copies {label}: " + " ".join(f"{r:.1f}" for r in rates) + " GB/s")
