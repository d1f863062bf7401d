"""CPU oracle (test infrastructure only; see oracle/engine.py header)."""
