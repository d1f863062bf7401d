"""Run the reference's unit and acceptance tests with the B200 engine installed.

    python tools/run_reference_suite.py [pytest args...]

Uses the unmodified reference installed by tools/reference_install.py
(baseline/_ref: the ``randbc`` package and a copy of its ``tests/`` and
``artifacts/``).  ``tools/rbc_dropin_plugin.py`` assigns
``paper_1905_07439_b200.engine.apply_levels`` / ``leaf_matmul`` into
``randbc._engine`` before collection, so every reference caller multiplies on
the GPU.  tests/test_reference_suite_gpu.py runs this as a ``-m gpu`` test.
"""

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


def command(extra=()):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT), str(ROOT / "tools"),
                                         env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    # test_draw_uniformity_chi_square: 10^6 host plan draws, no engine use
    cmd = [sys.executable, "-m", "pytest", "-p", "no:cacheprovider", "-p", "rbc_dropin_plugin",
           str(REF / "pkg" / "tests"), "-q", "-k", "not chi_square", *extra]
    return cmd, env


def main():
    if not (REF / "pkg" / "tests").is_dir():
        print("baseline/_ref missing: run python tools/reference_install.py")
        return 2
    cmd, env = command(sys.argv[1:])
    return subprocess.call(cmd, env=env, cwd=str(REF / "pkg" / "tests"))


if __name__ == "__main__":
    sys.exit(main())
