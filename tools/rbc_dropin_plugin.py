"""pytest plugin: route the reference's engine through the B200 engine.

Loaded with ``-p rbc_dropin_plugin`` when running the reference's own test
suite (tools/run_reference_suite.py).  Every call of
randbc._engine.apply_levels / leaf_matmul goes to paper_1905_07439_b200.engine;
calls in the decimal toy mode (out of scope for the GPU engine) skip the
calling test instead of falling back to numpy.
"""

import pytest

CALLS = {"apply_levels": 0, "leaf_matmul": 0, "skipped_decimal": 0}


def _wrap(fn, name):
    def call(*args, **kwargs):
        mode = kwargs.get("mode", args[3] if name == "apply_levels" and len(args) > 3 else
                          args[2] if name == "leaf_matmul" and len(args) > 2 else None)
        if getattr(mode, "kind", None) == "decimal":
            CALLS["skipped_decimal"] += 1
            pytest.skip("decimal toy machine is out of scope for the GPU engine")
        CALLS[name] += 1
        return fn(*args, **kwargs)

    return call


def pytest_configure(config):
    import randbc._engine as ref_engine

    from paper_1905_07439_b200 import _lib, engine

    _lib.require_device()
    ref_engine.apply_levels = _wrap(engine.apply_levels, "apply_levels")
    ref_engine.leaf_matmul = _wrap(engine.leaf_matmul, "leaf_matmul")


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"[drop-in] GPU engine calls: {CALLS}")
