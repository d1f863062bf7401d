"""cProfile of the reference's s2-variants run through the drop-in (GPU box):
where the wall clock of the reference user's workflow goes.
    python tools/dropin_profile.py [top]"""
import contextlib
import cProfile
import io
import pstats
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))

import randbc._engine  # noqa: E402
import randbc.cli  # noqa: E402

from paper_1905_07439_b200 import engine  # noqa: E402

engine.install(randbc._engine, wide="--wide" in sys.argv)
top = int(next((a for a in sys.argv[1:] if a.isdigit()), 35))
with tempfile.TemporaryDirectory() as d:
    out = Path(d) / "s2.csv"
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    with contextlib.redirect_stdout(io.StringIO()):
        pr.enable()
        code = randbc.cli.main(["experiment", "s2-variants", "--seed", "1", "--out", str(out)])
        pr.disable()
    print(f"exit {code}, {time.perf_counter() - t0:.2f} s")
    pstats.Stats(pr).sort_stats("cumulative").print_stats(top)
    pstats.Stats(pr).sort_stats("tottime").print_stats(20)
