"""Generate paper_1905_07439_b200/csrc/formulas_gen.cuh.

For every exact formula whose coefficients are in {-1, 0, +1} (Strassen,
Laderman, standard(2), standard(3)) this emits three straight-line device
networks in the formula's *base* coordinates:

  expand_u / expand_v : child_r = sum_kl c[r,k,l] * G[k][l]
  contract_w          : C[i][j] = sum_r w[r,i,j] * P_r

where G is the parent grid already gathered through the plan's signed
permutation (so the network itself is plan independent).  The rounding
sequence is the reference's (pkg/src/randbc/_engine.py:77-89, 104-112):

* a coefficient of +-1 makes the product exact, so a term is +-G;
* zero coefficients only add exact zeros and are dropped (values are equal
  to the reference's; only the sign of an exactly-zero result may differ);
* the row fold (over l) and the fold of row sums (over k) run in *hatted*
  order.  With n <= 3 a fold has at most three non-zero operands; for two
  the order is irrelevant (IEEE addition commutes), for three only the
  operand added last matters, and that is the base index sitting at hatted
  position n-1, i.e. perm[n-1] -- passed in at run time (lastrow/lastcol);
* the contraction folds over r ascending, which randomization never
  reorders, so it is fully static.  Signs are tracked symbolically
  (fl(-a - b) = -fl(a + b), fl(a - b) exact mirror) so no extra negations
  are emitted inside a chain.
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1905_07439_b200.formula import (  # noqa: E402
    laderman_formula,
    standard_formula,
    strassen_formula,
)

FORMULAS = [
    ("Strassen", 1, strassen_formula()),
    ("Laderman", 2, laderman_formula()),
    ("Standard2", 3, standard_formula(2)),
    ("Standard3", 4, standard_formula(3)),
]


class Emitter:
    def __init__(self):
        self.lines = []
        self.tmp = 0

    def new(self, expr):
        name = f"t{self.tmp}"
        self.tmp += 1
        self.lines.append(f"    const P {name} = {expr};")
        return name

    @staticmethod
    def combine(a, b, em):
        (sa, ea), (sb, eb) = a, b
        if sa == sb:
            return sa, em.new(f"O::add({ea}, {eb})")
        return sa, em.new(f"O::sub({ea}, {eb})")

    def materialize(self, x):
        s, e = x
        return e if s > 0 else self.new(f"O::neg({e})")


def expand_body(t, n, lastrow, lastcol):
    em = Emitter()
    outs = []
    for r in range(t.shape[0]):
        rows = []
        for k in range(n):
            elems = [(int(np.sign(t[r, k, l])), f"g[{k * n + l}]") for l in range(n) if t[r, k, l] != 0]
            for l in range(n):
                c = t[r, k, l]
                assert c in (0.0, 1.0, -1.0), "only +-1 formulas are code-generated"
            if not elems:
                continue
            if len(elems) == 1:
                rows.append(elems[0])
            elif len(elems) == 2:
                rows.append(Emitter.combine(elems[0], elems[1], em))
            else:
                assert len(elems) == 3
                xs = [em.materialize(x) for x in elems]
                rows.append((1, em.new(f"fold3<T, W>({xs[0]}, {xs[1]}, {xs[2]}, {lastcol})")))
        if not rows:
            outs.append("O::flip(g[0], 0) /* no terms */")
            em.lines.append(f"    o[{r}] = O::sub(g[0], g[0]);")
            continue
        if len(rows) == 1:
            acc = rows[0]
        elif len(rows) == 2:
            acc = Emitter.combine(rows[0], rows[1], em)
        else:
            assert len(rows) == 3
            xs = [em.materialize(x) for x in rows]
            acc = (1, em.new(f"fold3<T, W>({xs[0]}, {xs[1]}, {xs[2]}, {lastrow})"))
        s, e = acc
        em.lines.append(f"    o[{r}] = {e if s > 0 else f'O::neg({e})'};")
    return em.lines


def expand_one_body(t, n, r, lastrow, lastcol):
    """Output r alone of expand_body (same operations, same order)."""
    lines = expand_body(t[r:r + 1], n, lastrow, lastcol)
    return [ln.replace("o[0] = ", "return ") for ln in lines]


def contract_stream(w, n):
    """contract_body as a stream over r: per r, the accumulator updates that
    contract_body's chains perform for term r (acc holds sign * value), and
    the final sign fix-ups.  Same operations in the same order."""
    R = w.shape[0]
    sign = {}
    steps = []
    for r in range(R):
        lines = []
        for i in range(n):
            for j in range(n):
                c = w[r, i, j]
                if c == 0:
                    continue
                k = i * n + j
                st = int(np.sign(c))
                if k not in sign:
                    sign[k] = st
                    lines.append(f"        acc[{k}] = p;")
                elif sign[k] == st:
                    lines.append(f"        acc[{k}] = O::add(acc[{k}], p);")
                else:
                    lines.append(f"        acc[{k}] = O::sub(acc[{k}], p);")
        steps.append(lines)
    assert len(sign) == n * n, "streamed contraction needs a term for every output"
    finish = [f"    acc[{k}] = O::neg(acc[{k}]);" for k in sorted(sign) if sign[k] < 0]
    return steps, finish


def contract_body(w, n):
    em = Emitter()
    R = w.shape[0]
    for i in range(n):
        for j in range(n):
            acc = None
            for r in range(R):
                c = w[r, i, j]
                assert c in (0.0, 1.0, -1.0)
                if c == 0:
                    continue
                term = (int(np.sign(c)), f"p[{r}]")
                acc = term if acc is None else Emitter.combine(acc, term, em)
            if acc is None:
                em.lines.append(f"    o[{i * n + j}] = O::sub(p[0], p[0]);")
                continue
            s, e = acc
            em.lines.append(f"    o[{i * n + j}] = {e if s > 0 else f'O::neg({e})'};")
    return em.lines


def emit():
    out = [
        "// GENERATED by tools/gen_formulas.py -- do not edit.",
        "// Straight-line combination networks for exact +-1 bilinear formulas.",
        "#pragma once",
        '#include "common.cuh"',
        "",
        "namespace rbc {",
        "",
    ]
    ids = []
    for name, fid, f in FORMULAS:
        n, R = f.n, f.rank
        ids.append((name, fid))
        nnz = [int(np.count_nonzero(getattr(f, x))) for x in "uvw"]
        out.append(f"// {name}: n={n} R={R} nonzeros u/v/w = {nnz}")
        out.append(f"struct F{name} {{")
        out.append(f"  static constexpr int kId = {fid};")
        out.append(f"  static constexpr int n = {n};")
        out.append(f"  static constexpr int R = {R};")
        for tname, tensor in (("expand_u", f.u), ("expand_v", f.v)):
            out.append("  template <class T, int W>")
            out.append(
                f"  __device__ __forceinline__ static void {tname}("
                "const Pack<T, W>* g, Pack<T, W>* o, int lastrow, int lastcol) {"
            )
            out.append("    using P = Pack<T, W>;")
            out.append("    using O = PackOps<T, W>;")
            out.append("    (void)lastrow; (void)lastcol;")
            out.extend(expand_body(tensor, n, "lastrow", "lastcol"))
            out.append("  }")
        for mname, tensor in (("kU1Last", f.u), ("kV1Last", f.v)):
            # outputs whose single-output network has a runtime-ordered 3-term
            # fold (reads lastrow / lastcol); callers may specialise those
            mask = 0
            for r in range(R):
                if any("fold3" in ln for ln in expand_one_body(tensor, n, r, "lastrow", "lastcol")):
                    mask |= 1 << r
            out.append(f"  static constexpr unsigned long long {mname} = {mask:#x}ull;")
        for tname, tensor in (("expand_u1", f.u), ("expand_v1", f.v)):
            out.append("  // output r alone (r a compile-time constant after unrolling)")
            out.append("  template <class T, int W>")
            out.append(
                f"  __device__ __forceinline__ static Pack<T, W> {tname}("
                "const Pack<T, W>* g, int r, int lastrow, int lastcol) {"
            )
            out.append("    using P = Pack<T, W>;")
            out.append("    using O = PackOps<T, W>;")
            out.append("    (void)lastrow; (void)lastcol;")
            out.append("    switch (r) {")
            for r in range(R):
                out.append(f"      case {r}: {{")
                out.extend("  " + ln for ln in expand_one_body(tensor, n, r, "lastrow", "lastcol"))
                out.append("      }")
            out.append("      default: return g[0];")
            out.append("    }")
            out.append("  }")
        steps, finish = contract_stream(f.w, n)
        out.append("  // contract_w streamed over r ascending: step(r) for r = 0..R-1, then finish")
        out.append("  template <class T, int W>")
        out.append(
            "  __device__ __forceinline__ static void contract_w_step(Pack<T, W>* acc, "
            "const Pack<T, W>& p, int r) {"
        )
        out.append("    using O = PackOps<T, W>;")
        out.append("    switch (r) {")
        for r, lines in enumerate(steps):
            out.append(f"      case {r}:")
            out.extend(lines)
            out.append("        break;")
        out.append("      default: break;")
        out.append("    }")
        out.append("    (void)sizeof(O);")
        out.append("  }")
        out.append("  template <class T, int W>")
        out.append("  __device__ __forceinline__ static void contract_w_finish(Pack<T, W>* acc) {")
        out.append("    using O = PackOps<T, W>;")
        out.extend(finish)
        out.append("    (void)acc; (void)sizeof(O);")
        out.append("  }")
        out.append("  template <class T, int W>")
        out.append(
            "  __device__ __forceinline__ static void contract_w(const Pack<T, W>* p, Pack<T, W>* o) {"
        )
        out.append("    using P = Pack<T, W>;")
        out.append("    using O = PackOps<T, W>;")
        out.extend(contract_body(f.w, n))
        out.append("  }")
        out.append("};")
        out.append("")
    out.append("}  // namespace rbc")
    out.append("")
    out.append("// formula ids shared with the host (include/rbc.h RBC_FORMULA_*)")
    for name, fid in ids:
        out.append(f"#define RBC_GEN_FORMULA_{name.upper()} {fid}")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    path = ROOT / "paper_1905_07439_b200" / "csrc" / "formulas_gen.cuh"
    path.write_text(emit())
    print(f"wrote {path}")
