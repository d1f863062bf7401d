"""Device vs host generation of the BASELINE configs' seeded operand pairs.

    python tools/matgen_bench.py            (GPU box; prints one JSON line per config)
"""
import json
import sys
import time
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1905_07439_b200.configs import get_config, make_pairs, make_pairs_device  # noqa: E402

CASES = [("c1", 100, 100), ("c2", 1000, 100), ("c3", 4, 4), ("c4", 16, 2), ("c5", 2, 1)]


def main():
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    for name, pairs, host_pairs in CASES:
        if only and name != only:
            continue
        cfg = get_config(name)
        make_pairs_device(cfg, 1, min(pairs, 2))  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A, B = make_pairs_device(cfg, 1, pairs)
        torch.cuda.synchronize()
        dev_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        hA, hB = make_pairs(cfg, 1, host_pairs)
        host_s = (time.perf_counter() - t0) * pairs / host_pairs
        ok = (A[:host_pairs].cpu().numpy().tobytes() == hA.tobytes()
              and B[:host_pairs].cpu().numpy().tobytes() == hB.tobytes())
        elems = 2 * pairs * cfg.N * cfg.N
        print(json.dumps({"config": name, "kind": cfg.kind, "N": cfg.N, "pairs": pairs,
                          "device_ms": round(dev_s * 1e3, 3), "host_numpy_ms": round(host_s * 1e3, 1),
                          "host_sample_pairs": host_pairs, "speedup": round(host_s / dev_s, 1),
                          "device_gsamples_per_s": round(elems / dev_s / 1e9, 3),
                          "bitwise_equal_on_sample": ok}), flush=True)
        del A, B


if __name__ == "__main__":
    main()
