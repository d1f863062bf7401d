"""Run the reference's unit tests with the B200 engine installed.

    python tools/run_reference_suite.py [--prepare] [pytest args...]

--prepare copies /root/reference/pkg to baseline/_ref/pkg (git-ignored; it
travels to the GPU box with the repo snapshot).  Development aid only: the
product, tests/, smoke() and bench.py never use the reference.
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
COPY = ROOT / "baseline" / "_ref" / "pkg"


def main():
    args = sys.argv[1:]
    if args and args[0] == "--prepare":
        if COPY.exists():
            shutil.rmtree(COPY)
        shutil.copytree("/root/reference/pkg", COPY,
                        ignore=shutil.ignore_patterns("__pycache__", "*.pyc", "plots"))
        print(f"copied reference package to {COPY}")
        return 0
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(COPY / "src"), str(ROOT), str(ROOT / "tools"),
                                         env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-p", "no:cacheprovider", "-p", "rbc_dropin_plugin",
           str(COPY / "tests"), "-q", "-k", "not chi_square", *args]
    return subprocess.call(cmd, env=env, cwd=str(COPY / "tests"))


if __name__ == "__main__":
    sys.exit(main())
