"""Time the exact-order leaf kernels through the C ABI (tuning aid, GPU).

    python tools/leaf_bench.py  [--tiles 128,64]
"""
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1905_07439_b200 import _lib  # noqa: E402

CASES = [  # (label, dtype_in, dtype_out, batch, m)
    ("c5 leaf f32 256", 1, 1, 2 * 1681, 256),
    ("c1 leaf f32 64", 1, 1, 49 * 400, 64),
    ("c4 leaf f16 128", 2, 2, 2401 * 16, 128),
    ("truth f64<-f32 243", 1, 0, 200, 243),
    ("truth f64<-f32 256", 1, 0, 100, 256),
    ("truth f64<-f64 256", 0, 0, 100, 256),
    ("truth f64<-f32 2048", 1, 0, 2, 2048),
    ("truth f64<-f16 2048", 2, 0, 2, 2048),
    ("truth f64<-f16 2048x16", 2, 0, 16, 2048),
    ("truth f64<-f32 8192", 1, 0, 1, 8192),
    ("truth f64<-f64 729", 0, 0, 8, 729),
    ("c3 leaf f64 27", 0, 0, 12167 * 16, 27),
]
TORCH = {0: torch.float64, 1: torch.float32, 2: torch.float16}


def main():
    lib = _lib.load()
    tiles = (sys.argv[sys.argv.index("--tiles") + 1].split(",") if "--tiles" in sys.argv else ["0"])
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    for label, di, do, batch, m in CASES:
        if only and only not in label:
            continue
        x = torch.randn(batch, m, m, device="cuda").to(TORCH[di])
        y = torch.randn(batch, m, m, device="cuda").to(TORCH[di])
        out = torch.empty(batch, m, m, device="cuda", dtype=TORCH[do])
        first = None
        for t in tiles:
            os.environ["RBC_LEAF_TILE"] = t
            st = torch.cuda.current_stream()
            def run():
                rc = lib.rbc_leaf_matmul_async(di, do, batch, m * m, m * m, m, m, m,
                                               ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                               ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st.cuda_stream))
                _lib.check(rc)
            out.zero_()
            run(); torch.cuda.synchronize()
            if first is None:
                first = out.clone()
            same = torch.equal(out.view(torch.uint8), first.view(torch.uint8))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                run()
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            tf = 2.0 * batch * m ** 3 / (ms / 1e3) / 1e12
            print(f"{label:24s} tile={t:>4s} {ms:9.3f} ms {tf:7.2f} TFLOP/s  bits==first:{same}", flush=True)


if __name__ == "__main__":
    main()
