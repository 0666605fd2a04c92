"""Randomised shape sweep on both engines against the oracle's defining sums:
odd sizes around the tile edges (64 / 256 columns, 16 / 128-byte k chunks),
k-slab boundaries, every INT8 modulus count (11-16, through int8_bits),
non-HPD fractions and the unfused path.  Tolerance 1e-10 (north star)."""

import numpy as np
import pytest

from oracle import brute
from paper_1611_00606_b200 import Dims, GpuPolicy, ProblemSpec, build_hs, generate, int8_moduli, rel_frob_error

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _cases(n, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        n_atoms = int(rng.integers(1, 6))
        n_l = int(rng.choice([1, 4, 9, 16, 25, 49, 81, 121]))
        n_g = int(rng.choice([1, 7, 63, 64, 65, 127, 255, 256, 257, 300, 511, 513]))
        frac = float(rng.choice([0.0, 0.5, 1.0]))
        out.append((n_atoms, n_l, n_g, frac, 1000 + i))
    return out


@pytest.mark.parametrize("n_atoms,n_l,n_g,frac,seed", _cases(24))
@pytest.mark.parametrize("engine", ["int8", "dmma"])
def test_random_shapes(n_atoms, n_l, n_g, frac, seed, engine):
    p = generate(ProblemSpec(Dims(n_atoms, n_l, n_g), seed=seed, nonhpd_fraction=frac))
    out = build_hs(p, GpuPolicy(engine=engine))
    # both engines at FP64 width: FP64-level agreement, far inside the north star's 1e-10
    assert rel_frob_error(out.h.matrix, brute.h_brute(p)) < 1e-13
    assert rel_frob_error(out.s.matrix, brute.s_brute(p)) < 1e-13
    out.h.check()
    out.s.check()


@pytest.mark.parametrize("bits", [30, 34, 38, 42, 46, 48])
def test_every_modulus_count(bits):
    # int8_bits selects the moduli count (11 .. 16) through the exactness rule
    p = generate(ProblemSpec(Dims(3, 49, 333), seed=bits, nonhpd_fraction=0.34))
    n_mod, b = int8_moduli(3 * 3 * 49, bits)
    out = build_hs(p, GpuPolicy(engine="int8", int8_bits=bits))
    tol = max(TOL, 64 * 2.0 ** -b)  # 30 bits is below the north star's accuracy on purpose
    assert rel_frob_error(out.h.matrix, brute.h_brute(p)) < tol, (n_mod, b)
    assert rel_frob_error(out.s.matrix, brute.s_brute(p)) < tol, (n_mod, b)


@pytest.mark.parametrize("fused", [True, False])
def test_slab_boundary_reductions(fused):
    # H's K_tot = 3 x 46 x 121 = 16698 bytes of k per residue row: two 16 KB slabs
    # (the second accumulates into the first in place); S stays single-slab
    p = generate(ProblemSpec(Dims(46, 121, 200), seed=5, nonhpd_fraction=0.25))
    out = build_hs(p, GpuPolicy(engine="int8", fused=fused))
    assert rel_frob_error(out.h.matrix, brute.h_brute(p)) < TOL
    assert rel_frob_error(out.s.matrix, brute.s_brute(p)) < TOL
