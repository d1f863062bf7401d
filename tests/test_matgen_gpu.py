"""GPU: seeded test matrices drawn on the device (librbc rbc_matgen) are
bit-identical to the reference's host draws -- numpy's Philox4x64 stream,
Generator.random() and Generator.standard_normal() (ziggurat, incl. its
wedge and tail paths) -- for every family, in every mode (
reference matgen.py:55-97, rng.py:20-23)."""

import numpy as np
import pytest

from paper_1905_07439_b200.matgen import BUILDER_KINDS, MATRIX_KINDS, MatrixSpec, generate
from paper_1905_07439_b200.precision import DOUBLE, HALF, SINGLE

pytestmark = pytest.mark.gpu


def _host(kind, n, seed, mode):
    A, B = generate(MatrixSpec(kind, n, seed))
    return mode.array(A), mode.array(B)


@pytest.mark.parametrize("kind", MATRIX_KINDS + BUILDER_KINDS)
@pytest.mark.parametrize("n", [1, 7, 64, 243])
def test_families_bitwise_f64(kind, n):
    from paper_1905_07439_b200.matgen import generate_device

    if kind.startswith("adv") and n < 2:
        pytest.skip("adversarial kinds need n >= 2")
    seeds = [3, 2**63 + 5, 17]
    A, B = generate_device(kind, n, seeds, DOUBLE)
    for c, sd in enumerate(seeds):
        a, b = _host(kind, n, sd, DOUBLE)
        assert A[c].cpu().numpy().tobytes() == a.tobytes(), (kind, n, sd, "A")
        assert B[c].cpu().numpy().tobytes() == b.tobytes(), (kind, n, sd, "B")


@pytest.mark.parametrize("mode,kind,n", [(SINGLE, "uniform_pm1", 243), (SINGLE, "gaussian", 256),
                                         (HALF, "quadrant100", 512), (SINGLE, "adv1", 320)])
def test_mode_rounding_bitwise(mode, kind, n):
    from paper_1905_07439_b200.matgen import generate_device

    seeds = [11, 12]
    A, B = generate_device(kind, n, seeds, mode)
    for c, sd in enumerate(seeds):
        a, b = _host(kind, n, sd, mode)
        assert A[c].cpu().numpy().tobytes() == a.tobytes()
        assert B[c].cpu().numpy().tobytes() == b.tobytes()


def test_long_normal_stream_bitwise():
    """4M normals per stream: ~1000 tail samples and ~50K wedge tests each."""
    from paper_1905_07439_b200.matgen import generate_device

    n = 2048
    seeds = [99, 100]
    (A,) = generate_device("gaussian", n, seeds, DOUBLE, which=(0,))
    for c, sd in enumerate(seeds):
        a, _ = generate(MatrixSpec("gaussian", n, sd))
        got = A[c].cpu().numpy()
        bad = int(np.sum(got != a))
        assert bad == 0, f"{bad} of {a.size} samples differ"


def test_half_overflow_raises():
    """Uniform * n^2 (adv2's huge block) overflows binary16 like mode.array."""
    from paper_1905_07439_b200.matgen import generate_device

    with pytest.raises(OverflowError):
        _host("adv2", 512, 5, HALF)
    with pytest.raises(OverflowError):
        generate_device("adv2", 512, [5], HALF)


def test_config_pairs_device_match_host():
    from dataclasses import replace

    from paper_1905_07439_b200.configs import get_config, make_pairs, make_pairs_device

    for name, N in (("c2", 243), ("c4", 256), ("c3", 81)):
        cfg = replace(get_config(name), N=N)
        A, B = make_pairs(cfg, 3, 2)
        dA, dB = make_pairs_device(cfg, 3, 2)
        assert dA.cpu().numpy().tobytes() == A.tobytes()
        assert dB.cpu().numpy().tobytes() == B.tobytes()
