"""Time the parts of one fresh-input error-trial step (GPU box):
    python tools/fresh_probe.py [config] [pairs]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1905_07439_b200.configs import get_config, make_pairs_device, packed_plans, pair_seeds  # noqa: E402
from paper_1905_07439_b200.trials import DeviceErrorTrials  # noqa: E402


def main():
    cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    dev = torch.device("cuda:0")
    r = DeviceErrorTrials(cfg.formula_obj(), cfg.Q, cfg.N, cfg.mode, T, device=dev)
    p0 = 1
    for it in range(6):
        t = [time.perf_counter()]
        s = pair_seeds(cfg, p0, T); t.append(time.perf_counter())
        a, b = make_pairs_device(cfg, p0, T, dev); torch.cuda.synchronize(); t.append(time.perf_counter())
        pl = torch.from_numpy(packed_plans(cfg, [cfg.plan_key(p) for p in range(p0, p0 + T)])); t.append(time.perf_counter())
        pl = pl.to(dev); t.append(time.perf_counter())
        r.run(a, b, pl); t.append(time.perf_counter())
        torch.cuda.synchronize(); t.append(time.perf_counter())
        e = r.err_rand.cpu(); t.append(time.perf_counter())
        names = ["seeds", "matgen", "plans", "h2d", "enqueue", "compute", "d2h"]
        print(" ".join(f"{n}={1e3 * (t[i + 1] - t[i]):.2f}" for i, n in enumerate(names)),
              f"total={1e3 * (t[-1] - t[0]):.2f} ms", flush=True)
        p0 += T
        del s, e


if __name__ == "__main__":
    main()
