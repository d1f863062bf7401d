"""Install the unmodified reference (`randbc`) into baseline/_ref.

    python tools/reference_install.py [--force]

Test and benchmark infrastructure only (the product never imports it):

* ``baseline/_ref/randbc``      -- ``pip install --no-index --no-deps --target``
  of a /tmp copy of /root/reference/pkg (the source tree is read-only), the
  unmodified reference package; ``bench.py --impl reference`` times it and
  ``tests/test_reference_suite_gpu.py`` drives its callers through the drop-in;
* ``baseline/_ref/pkg/tests``, ``baseline/_ref/pkg/artifacts`` -- the
  reference's own unit/acceptance suite and its artifact directory, run by
  ``tests/test_reference_suite_gpu.py`` with the B200 engine installed.

baseline/_ref is git-ignored but not gpurun-ignored, so it travels to the GPU
box with the repo snapshot; /root/reference itself does not exist there.
"""

from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF_SRC = Path("/root/reference/pkg")
TARGET = ROOT / "baseline" / "_ref"


def installed() -> bool:
    return (TARGET / "randbc" / "_engine.py").exists() and (TARGET / "pkg" / "tests").is_dir()


def ensure(force: bool = False) -> bool:
    """Install when missing (or forced) and the reference tree is present.
    Returns whether baseline/_ref holds the reference afterwards."""
    if installed() and not force:
        return True
    if not REF_SRC.is_dir():
        return installed()
    TARGET.mkdir(parents=True, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REF_SRC, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
        for old in TARGET.glob("randbc*"):
            shutil.rmtree(old) if old.is_dir() else old.unlink()
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--find-links", "/opt/wheelhouse", "--target", str(TARGET),
               "--upgrade", str(src)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"reference install failed:\n{res.stdout}\n{res.stderr}")
    pkg = TARGET / "pkg"
    if pkg.exists():
        shutil.rmtree(pkg)
    pkg.mkdir()
    for sub in ("tests", "artifacts"):
        shutil.copytree(REF_SRC / sub, pkg / sub,
                        ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    return installed()


if __name__ == "__main__":
    ok = ensure(force="--force" in sys.argv)
    print(f"baseline/_ref: {'installed' if ok else 'unavailable'}")
    sys.exit(0 if ok else 1)
