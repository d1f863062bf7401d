"""CPU oracle (test infrastructure only) of the device matrix generator --
pure-Python restatement of the algorithm librbc's matgen.cu runs, step for
step, for pinning it against numpy (the reference's generator).

Reference: derive_rng / matgen.generate (pkg/src/randbc/rng.py:20-23,
matgen.py:55-97) draw from numpy's Generator(Philox(SeedSequence)).  numpy is
a third-party dependency (pinned numpy>=1.24, pkg/pyproject.toml:12; numpy 2.3
in this image); its published algorithms are restated here:

* Philox4x64-10 (Salmon, Moraes, Dror, Shaw, SC'11): 10 rounds of two 64x64
  multiplies with the Weyl key schedule; numpy's stream word i is lane i % 4
  of the block at counter (i // 4 + 1, 0, 0, 0).
* Generator.random(): (word >> 11) * 2**-53.
* Generator.standard_normal(): Marsaglia-Tsang ziggurat with 256 strips as
  numpy formulates it (strip index = low byte, sign = bit 8, 52-bit magnitude
  above; fast accept below ki[idx]; strip 0 -> exponential tail; else wedge
  test against exp(-x*x/2)), with numpy's tables -- the build reads them from
  numpy's shipped libnpyrandom.a into build/gen/ziggurat_tables.inc, which is
  parsed here.

Pinning: tests/test_oracle_matgen.py checks this restatement against numpy's
own Philox.random_raw / Generator.random / Generator.standard_normal.  Only
tests, __graft_entry__.smoke() and bench.py's cpu_baseline may import this.
"""

from __future__ import annotations

import math
import re
from pathlib import Path

import numpy as np

MASK = (1 << 64) - 1
M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
ZIG_R = 3.6541528853610088
ZIG_INV_R = 0.27366123732975828

_TABLES = None


def philox4x64_10(ctr, key):
    c = list(ctr)
    k0, k1 = key
    for _ in range(10):
        p0, p1 = M0 * c[0], M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k0, p1 & MASK, (p0 >> 64) ^ c[3] ^ k1, p0 & MASK]
        k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
    return c


def raw_words(key, count: int) -> list[int]:
    out = []
    for blk in range((count + 3) // 4):
        out += philox4x64_10([blk + 1, 0, 0, 0], key)
    return out[:count]


def unit_double(w: int) -> float:
    return (w >> 11) * (1.0 / 9007199254740992.0)


def tables():
    """(ki, wi, fi) parsed from the generated header of the last build."""
    global _TABLES
    if _TABLES is None:
        hdr = Path(__file__).resolve().parents[1] / "paper_1905_07439_b200" / "build" / "gen" / "ziggurat_tables.inc"
        if not hdr.exists():
            from paper_1905_07439_b200.build import _ziggurat_header

            _ziggurat_header()
        txt = hdr.read_text()

        def grab(name):
            return re.search(rf"{name} \{{(.*)\}}", txt).group(1).split(", ")

        ki = [int(v.rstrip("ul"), 16) for v in grab("RBC_ZIG_KI")]
        wi = [float.fromhex(v) for v in grab("RBC_ZIG_WI")]
        fi = [float.fromhex(v) for v in grab("RBC_ZIG_FI")]
        _TABLES = (ki, wi, fi)
    return _TABLES


def standard_normals(words, n: int) -> np.ndarray:
    """The first n standard normals of a raw word stream."""
    ki, wi, fi = tables()
    it = iter(words)
    out = []
    while len(out) < n:
        r = next(it)
        idx = r & 0xFF
        rabs = (r >> 9) & 0x000FFFFFFFFFFFFF
        x = float(rabs) * wi[idx]
        if (r >> 8) & 1:
            x = -x
        if rabs < ki[idx]:
            out.append(x)
        elif idx == 0:
            while True:
                xx = -ZIG_INV_R * math.log1p(-unit_double(next(it)))
                yy = -math.log1p(-unit_double(next(it)))
                if yy + yy > xx * xx:
                    out.append(-(ZIG_R + xx) if (rabs >> 8) & 1 else ZIG_R + xx)
                    break
        elif (fi[idx - 1] - fi[idx]) * unit_double(next(it)) + fi[idx] < math.exp(-0.5 * x * x):
            out.append(x)
    return np.array(out)
