"""B200-native randomized bilinear-computation (BC) matrix multiply.

A from-scratch sm_100a implementation of the hot path of arXiv 1905.07439's
reference package ``randbc``: the breadth-first recursive evaluation of
C = AB from (U, V, W) under per-level random signed permutations.

Public surface (mirrors the reference's names and semantics):

* engine boundary : ``engine.apply_levels``, ``engine.leaf_matmul``,
                    ``engine.install`` (patches ``randbc._engine``)
* north star      : ``bc_matmul(A, B, U, V, W, depth, randomize, seed, dtype)``
* L2 API          : ``standard_multiply``, ``apply_bc``, ``recursive_apply``,
                    ``randomized_apply``, ``recursive_randomized_apply[_many]``
* formulas/plans  : ``BilinearFormula``, ``strassen_formula``,
                    ``laderman_formula``, ``perturb``, ``perturb_all``,
                    ``kappa``, ``draw_plan``, ``hatted_tensors`` ...
* modes           : ``DOUBLE``, ``SINGLE``, ``HALF``
* device pipeline : ``trials`` (ground truth + relative errors on device)
"""

from .formula import (
    BilinearFormula,
    format_formula,
    is_exact,
    kappa,
    laderman_formula,
    load_formula,
    parse_formula,
    perturb,
    perturb_all,
    save_formula,
    standard_formula,
    strassen_formula,
)
from .matgen import MATRIX_KINDS, MatrixSpec, generate
from .multiply import apply_bc, bc_matmul, mode_tensors, recursive_apply, standard_multiply
from .precision import DOUBLE, HALF, SINGLE, Mode, parse_precision
from .randomize import (
    VARIANTS,
    RandomizationPlan,
    RecursivePlan,
    draw_plan,
    draw_recursive_plan,
    hatted_tensors,
    identity_plan,
    identity_recursive_plan,
    plan_levels,
    randomized_apply,
    recursive_randomized_apply,
    recursive_randomized_apply_many,
    variant_plan,
)
from .rng import ROLE_FORMULA, ROLE_INPUT, ROLE_MATRIX, ROLE_PLAN, derive_rng, derive_seed

__version__ = "0.1.0"
