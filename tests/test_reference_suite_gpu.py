"""The reference's own test suite, run with the B200 engine as its drop-in.

The unmodified reference (baseline/_ref, installed by
tools/reference_install.py) runs its unit and acceptance tests -- including
the full-scale ``randbc experiment s2-variants`` replication at n=320
(reference pkg/tests/test_acceptance.py:330-365) -- with
``randbc._engine.apply_levels`` / ``leaf_matmul`` assigned to
``paper_1905_07439_b200.engine`` (tools/rbc_dropin_plugin.py).  Tests that
drive the engine in the decimal toy mode (out of scope) are skipped by the
plugin, never run on numpy.  Skipped when baseline/_ref is absent.
"""

import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not (REF / "pkg" / "tests").is_dir(), reason="baseline/_ref not installed")
def test_reference_suite_through_dropin():
    from paper_1905_07439_b200 import _lib

    _lib.require_device()
    sys.path.insert(0, str(ROOT / "tools"))
    try:
        import run_reference_suite
    finally:
        sys.path.pop(0)
    cmd, env = run_reference_suite.command()
    res = subprocess.run(cmd, env=env, cwd=str(REF / "pkg" / "tests"), capture_output=True,
                         text=True, timeout=900)
    tail = (res.stdout + res.stderr)[-3000:]
    assert res.returncode == 0, tail
    m = re.search(r"\[drop-in\] GPU engine calls: \{'apply_levels': (\d+), 'leaf_matmul': (\d+)", tail)
    assert m, tail
    assert int(m.group(1)) > 1000 and int(m.group(2)) > 100, tail
    summary = re.search(r"(\d+) passed", tail)
    assert summary and int(summary.group(1)) >= 250, tail
    print(tail[-600:])
