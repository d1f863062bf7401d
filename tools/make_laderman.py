"""Write paper_1905_07439_b200/formulas/laderman.txt.

Laderman, "A noncommutative algorithm for multiplying 3x3 matrices using 23
multiplications", Bull. AMS 82 (1976) -- cited by the paper at PAPER.md:27.
The 23 products m1..m23 are entered below as signed sums of 1-based block
names; the file is validated with is_exact() and kappa() == 0 before writing.
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1905_07439_b200.formula import (  # noqa: E402
    BilinearFormula,
    format_formula,
    is_exact,
    kappa,
)

# (A combination, B combination) per product; "-21" means -A21 / -B21.
PRODUCTS = [
    ("11 12 13 -21 -22 -32 -33", "22"),
    ("11 -21", "-12 22"),
    ("22", "-11 12 21 -22 -23 -31 33"),
    ("-11 21 22", "11 -12 22"),
    ("21 22", "-11 12"),
    ("11", "11"),
    ("-11 31 32", "11 -13 23"),
    ("-11 31", "13 -23"),
    ("31 32", "-11 13"),
    ("11 12 13 -22 -23 -31 -32", "23"),
    ("32", "-11 13 21 -22 -23 -31 32"),
    ("-13 32 33", "22 31 -32"),
    ("13 -33", "22 -32"),
    ("13", "31"),
    ("32 33", "-31 32"),
    ("-13 22 23", "23 31 -33"),
    ("13 -23", "23 -33"),
    ("22 23", "-31 33"),
    ("12", "21"),
    ("23", "32"),
    ("21", "13"),
    ("31", "12"),
    ("33", "33"),
]

# C block -> 1-based products summed into it
OUTPUTS = {
    "11": (6, 14, 19),
    "12": (1, 4, 5, 6, 12, 14, 15),
    "13": (6, 7, 9, 10, 14, 16, 18),
    "21": (2, 3, 4, 6, 14, 16, 17),
    "22": (2, 4, 5, 6, 20),
    "23": (14, 16, 17, 18, 21),
    "31": (6, 7, 8, 11, 12, 13, 14),
    "32": (12, 13, 14, 15, 22),
    "33": (6, 7, 8, 9, 23),
}


def _fill(t, r, spec):
    for tok in spec.split():
        sign = -1.0 if tok.startswith("-") else 1.0
        name = tok.lstrip("-")
        t[r, int(name[0]) - 1, int(name[1]) - 1] = sign


def build() -> BilinearFormula:
    u = np.zeros((23, 3, 3))
    v = np.zeros((23, 3, 3))
    w = np.zeros((23, 3, 3))
    for r, (a, b) in enumerate(PRODUCTS):
        _fill(u, r, a)
        _fill(v, r, b)
    for name, rs in OUTPUTS.items():
        for r in rs:
            w[r - 1, int(name[0]) - 1, int(name[1]) - 1] = 1.0
    return BilinearFormula(u, v, w)


if __name__ == "__main__":
    f = build()
    assert is_exact(f, 0.0) and kappa(f) == 0.0
    out = ROOT / "paper_1905_07439_b200" / "formulas" / "laderman.txt"
    out.write_text(format_formula(f), encoding="ascii")
    print(f"wrote {out}")
