"""The C ABI from plain C: include/rbc.h compiles as C99 and a C client links
against librbc.so (CPU check); on a GPU the client's leaf product and
two-level Strassen product equal their C restatements bit for bit."""
import os
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_1905_07439_b200" / "lib"


def _build(tmp_path):
    from paper_1905_07439_b200 import _lib

    _lib.load()  # builds the library if needed
    exe = tmp_path / "capi_client"
    cmd = [shutil.which("gcc") or "gcc", "-std=c99", "-O1", "-ffp-contract=off", "-Wall", "-Werror",
           f"-I{ROOT / 'include'}", str(ROOT / "tests" / "capi" / "capi_client.c"),
           f"-L{LIBDIR}", "-lrbc", "-lm", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return exe


def test_header_is_c99_and_client_links(tmp_path):
    exe = _build(tmp_path)
    assert exe.exists()
    # every rbc_ symbol the client references resolves against librbc.so
    nm = subprocess.run(["nm", "-u", str(exe)], capture_output=True, text=True).stdout
    assert "rbc_apply_levels" in nm and "rbc_leaf_matmul" in nm


@pytest.mark.gpu
def test_c_client_runs_on_the_gpu(tmp_path):
    exe = _build(tmp_path)
    res = subprocess.run([str(exe)], capture_output=True, text=True, env=dict(os.environ))
    assert res.returncode == 0, res.stdout + res.stderr
    assert "capi client ok" in res.stdout
