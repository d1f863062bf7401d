"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the development container only (it imports ``randbc`` from
/root/reference/pkg/src, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Outputs (committed):
  engine_cases.npz / engine_cases.json  -- inputs, coefficient tables, plans and
      outputs of ``randbc._engine.apply_levels`` / ``leaf_matmul`` for a set of
      formulas, modes, depths and trial layouts (incl. an fp16 overflow case)
  host_cases.npz                         -- draw_plan / hatted_tensors / kappa /
      perturb / generate outputs, pinning the host-side mirror
  experiments_tiny.csv                   -- ``run_experiment`` records of small
      s2_variants / s1_dist configs (bitwise reproducible from the seed layout)
  s2_variants_320.csv                    -- the whole reference artifact
      pkg/artifacts/s2-variants-320.csv (seed 1, all six families, 9066 rows)

binary16 goes through the unmodified reference engine with this package's
duck-typed HALF mode (parity against the reference is unpinned
for fp16 -- the reference has no fp16 -- but parity against the reference's
own engine arithmetic is bitwise).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import randbc  # noqa: E402
from randbc import _engine  # noqa: E402
from randbc.experiments import ExperimentConfig, format_csv, run_experiment  # noqa: E402
from randbc.formula import BilinearFormula, kappa, perturb, standard_formula, strassen_formula  # noqa: E402
from randbc.matgen import MatrixSpec, generate  # noqa: E402
from randbc.precision import DOUBLE, SINGLE  # noqa: E402
from randbc.randomize import _plan_levels, draw_plan, hatted_tensors  # noqa: E402
from randbc.rng import derive_rng, derive_seed  # noqa: E402

from paper_1905_07439_b200.formula import load_formula  # noqa: E402
from paper_1905_07439_b200.precision import HALF  # noqa: E402

LADERMAN_FILE = ROOT / "paper_1905_07439_b200" / "formulas" / "laderman.txt"


def laderman():
    g = load_formula(LADERMAN_FILE)
    return BilinearFormula(g.u, g.v, g.w)


def laderman_noisy(seed=1, sigma=1e-4):
    f = laderman()
    noise = derive_rng(seed, 0).normal(0.0, sigma, size=(3,) + f.u.shape)
    return BilinearFormula(f.u + noise[0], f.v + noise[1], f.w + noise[2])


FORMULAS = {
    "strassen": (strassen_formula, "strassen"),
    "perturbed": (lambda: perturb(strassen_formula(), 1e-3, 5, derive_rng(42)), None),
    "laderman": (laderman, "laderman"),
    "laderman_noisy": (laderman_noisy, None),
    "standard2": (lambda: standard_formula(2), "standard2"),
    "standard3": (lambda: standard_formula(3), "standard3"),
    "all_ones": (lambda: BilinearFormula(np.ones((1, 2, 2)), np.ones((1, 2, 2)), np.ones((1, 2, 2))), None),
}

MODES = {"f64": DOUBLE, "f32": SINGLE, "f16": HALF}

# name, formula, mode, Q, N, T0, plan layout ("det" = identity, Tc=1;
# "rand" = per-trial plans; "mixed" = identity level 0, per-trial deeper),
# T (plans), input kind
ENGINE_CASES = [
    ("E01_strassen_f32_rand", "strassen", "f32", 2, 8, 1, "rand", 3, "gaussian"),
    ("E02_strassen_f64_det", "strassen", "f64", 3, 16, 1, "det", 1, "gaussian"),
    ("E03_perturbed_f64_rand", "perturbed", "f64", 2, 12, 1, "rand", 4, "gaussian"),
    ("E04_laderman_f32_rand", "laderman", "f32", 2, 18, 1, "rand", 3, "uniform_pm1"),
    ("E05_ladnoisy_f64_rand", "laderman_noisy", "f64", 2, 9, 1, "rand", 2, "gaussian"),
    ("E06_standard2_f32_det", "standard2", "f32", 2, 8, 1, "det", 1, "gaussian"),
    ("E07_allones_f64_raw", "all_ones", "f64", 1, 4, 1, "raw", 1, "gaussian"),
    ("E08_strassen_f16_rand", "strassen", "f16", 2, 16, 1, "rand", 3, "gaussian"),
    ("E09_strassen_f16_overflow", "strassen", "f16", 2, 16, 1, "det", 1, "quadrant1e3"),
    ("E10_strassen_f32_pairs", "strassen", "f32", 2, 8, 3, "rand", 3, "gaussian"),
    ("E11_laderman_f64_det", "laderman", "f64", 1, 3, 1, "det", 1, "gaussian"),
    ("E12_standard3_f32_det", "standard3", "f32", 1, 6, 1, "det", 1, "gaussian"),
    ("E13_strassen_f32_m1", "strassen", "f32", 3, 8, 1, "rand", 2, "gaussian"),
    ("E14_strassen_f32_mixed", "strassen", "f32", 2, 8, 1, "mixed", 3, "gaussian"),
    ("E15_laderman_f32_q3", "laderman", "f32", 3, 27, 1, "rand", 2, "uniform_pm1"),
    ("E16_perturbed_f32_rand", "perturbed", "f32", 3, 24, 1, "rand", 3, "gaussian"),
    ("E17_ladnoisy_f16_rand", "laderman_noisy", "f16", 1, 6, 1, "rand", 2, "gaussian"),
    ("E18_laderman_f16_rand", "laderman", "f16", 2, 18, 2, "rand", 2, "gaussian"),
    ("E19_strassen_f64_rand_q4", "strassen", "f64", 4, 48, 1, "rand", 2, "gaussian"),
    ("E20_strassen_f32_q1_m64", "strassen", "f32", 1, 128, 1, "rand", 2, "gaussian"),
]

LEAF_CASES = [
    ("L01_f64_rect", "f64", (1, 4, 6), (1, 6, 5)),
    ("L02_f32_broadcast", "f32", (3, 1, 4, 5), (2, 5, 3)),
    ("L03_f64_empty_k", "f64", (2, 3, 0), (2, 0, 4)),
    ("L04_f32_tile64", "f32", (2, 70, 70), (2, 70, 70)),
    ("L05_f32_tile128", "f32", (1, 130, 131), (1, 131, 129)),
    ("L06_f64_tile32", "f64", (2, 40, 33), (2, 33, 41)),
    ("L07_f16_small", "f16", (2, 9, 7), (2, 7, 5)),
    ("L08_f64_tile64", "f64", (1, 96, 100), (1, 100, 80)),
    ("L09_f16_tile", "f16", (1, 70, 66), (1, 66, 72)),
]


def operands(kind, N, T0, seed):
    out_a, out_b = [], []
    for t in range(T0):
        ga, gb = derive_rng(seed, 0, t), derive_rng(seed, 1, t)
        if kind == "gaussian":
            A, B = ga.standard_normal((N, N)), gb.standard_normal((N, N))
        elif kind == "uniform_pm1":
            A, B = 2 * ga.random((N, N)) - 1, 2 * gb.random((N, N)) - 1
        elif kind == "quadrant1e3":
            A, B = ga.standard_normal((N, N)), gb.standard_normal((N, N))
            A[: N // 2, : N // 2] *= 1e3
            B[N // 2 :, N // 2 :] *= 1e3
        else:
            raise ValueError(kind)
        out_a.append(A)
        out_b.append(B)
    return np.stack(out_a), np.stack(out_b)


def plans_for(layout, n, Q, T, seed):
    ident = (np.ones((3, n)), np.tile(np.arange(n), (3, 1)))
    perms = np.zeros((T if layout != "det" else 1, Q, 3, n), dtype=np.int64)
    signs = np.zeros(perms.shape)
    for t in range(perms.shape[0]):
        for q in range(Q):
            if layout == "det" or (layout == "mixed" and q == 0):
                s, p = ident
            else:
                pl = draw_plan(n, derive_rng(seed, 2, t, q))
                s, p = pl.signs, pl.perms
            perms[t, q] = p
            signs[t, q] = s
    return perms, signs


def main():
    arrays = {}
    meta = {"engine": [], "leaf": []}
    for idx, (name, fkey, mkey, Q, N, T0, layout, T, kind) in enumerate(ENGINE_CASES):
        f = FORMULAS[fkey][0]()
        mode = MODES[mkey]
        A64, B64 = operands(kind, N, T0, 1000 + idx)
        a, b = mode.array(A64), mode.array(B64)
        if layout == "raw":
            levels = [tuple(mode.array(t)[None] for t in (f.u, f.v, f.w))] * Q
            perms = signs = None
        else:
            perms, signs = plans_for(layout, f.n, Q, T, 2000 + idx)
            levels = []
            for q in range(Q):
                if layout == "mixed" and q == 0:
                    from randbc.randomize import RandomizationPlan

                    lv = _plan_levels(f, [RandomizationPlan(signs[0, q], perms[0, q])], mode)
                else:
                    from randbc.randomize import RandomizationPlan

                    lv = _plan_levels(
                        f, [RandomizationPlan(signs[t, q], perms[t, q]) for t in range(perms.shape[0])], mode
                    )
                levels.append(lv)
        stats = {}
        entry = {
            "name": name, "formula": fkey, "plan_formula": FORMULAS[fkey][1], "mode": mkey,
            "Q": Q, "N": N, "T0": T0, "layout": layout, "n": f.n, "R": f.rank,
        }
        try:
            out = _engine.apply_levels(levels, a, b, mode, stats)
            entry["raises"] = None
            arrays[f"{name}/out"] = out
            entry["leaf_multiplies"] = int(stats["leaf_multiplies"])
        except OverflowError as e:
            entry["raises"] = "OverflowError"
            entry["message"] = str(e)
        arrays[f"{name}/a"] = a
        arrays[f"{name}/b"] = b
        for q, (u, v, w) in enumerate(levels):
            arrays[f"{name}/u{q}"] = u
            arrays[f"{name}/v{q}"] = v
            arrays[f"{name}/w{q}"] = w
        if perms is not None:
            arrays[f"{name}/perms"] = perms
            arrays[f"{name}/signs"] = signs
        meta["engine"].append(entry)

    for idx, (name, mkey, xs, ys) in enumerate(LEAF_CASES):
        mode = MODES[mkey]
        g = derive_rng(3000 + idx)
        x = mode.array(g.standard_normal(xs))
        y = mode.array(g.standard_normal(ys))
        out = _engine.leaf_matmul(x, y, mode)
        arrays[f"{name}/x"] = x
        arrays[f"{name}/y"] = y
        arrays[f"{name}/out"] = out
        meta["leaf"].append({"name": name, "mode": mkey})
    # crafted order case (reference test_multiply.py:76-81)
    x = np.array([[[1.0, 1e-16, -1.0]]])
    y = np.array([[[1.0], [1.0], [1.0]]])
    arrays["L10_f64_order/x"] = x
    arrays["L10_f64_order/y"] = y
    arrays["L10_f64_order/out"] = _engine.leaf_matmul(x, y, DOUBLE)
    meta["leaf"].append({"name": "L10_f64_order", "mode": "f64"})

    np.savez_compressed(HERE / "engine_cases.npz", **arrays)
    (HERE / "engine_cases.json").write_text(json.dumps(meta, indent=1))

    # ---- host-side pins
    host = {}
    for seed in range(4):
        for n in (2, 3):
            p = draw_plan(n, derive_rng(seed, 2, seed + 1, n))
            host[f"plan/{seed}/{n}/signs"] = p.signs
            host[f"plan/{seed}/{n}/perms"] = p.perms
    f = perturb(strassen_formula(), 1e-3, 5, derive_rng(42))
    for x in "uvw":
        host[f"perturbed/{x}"] = getattr(f, x)
    host["perturbed/kappa"] = np.array(kappa(f))
    ln = laderman_noisy()
    host["laderman_noisy/kappa"] = np.array(kappa(ln))
    pl = draw_plan(2, derive_rng(9))
    for x, t in zip("uvw", hatted_tensors(f, pl)):
        host[f"hatted/{x}"] = t
    host["hatted/signs"] = pl.signs
    host["hatted/perms"] = pl.perms
    for kind in ("gaussian", "uniform", "adv1", "adv2", "adv3", "hilbert"):
        A, B = generate(MatrixSpec(kind, 6, derive_seed(1, 1, 0, 0)))
        host[f"matgen/{kind}/A"] = A
        host[f"matgen/{kind}/B"] = B
    host["derive_seed/1_1_0_0"] = np.array(derive_seed(1, 1, 0, 0), dtype=np.uint64)
    np.savez_compressed(HERE / "host_cases.npz", **host)

    # ---- experiment records (tiny configs)
    recs = []
    cfg = ExperimentConfig("s2_variants", "all", 32, 3, 4, 7, SINGLE)
    recs += run_experiment(cfg)
    cfg = ExperimentConfig("s1_dist", "gaussian", 16, 2, 3, 5, DOUBLE)
    recs += run_experiment(cfg)
    (HERE / "experiments_tiny.csv").write_text(format_csv(recs))

    # ---- the reference artifact (whole)
    src = Path("/root/reference/pkg/artifacts/s2-variants-320.csv").read_text().splitlines()
    # the whole artifact: all six matrix families (9066 rows)
    (HERE / "s2_variants_320.csv").write_text("\n".join(src) + "\n")
    keep = src
    print(f"engine cases: {len(meta['engine'])}, leaf cases: {len(meta['leaf'])}, "
          f"experiment rows: {len(recs)}, artifact rows: {len(keep) - 1}")


if __name__ == "__main__":
    main()
