"""Matching coefficients, CPU side: the G-vector set (host, shared by GPU and
oracle) and the oracle restatement's closed-form pins.  The reference has no
implementation of this row: these known answers are what pin
the oracle (parity unpinned by the reference)."""

import math

import numpy as np
import pytest
import scipy.special as sp

from oracle import matching as om
from paper_1611_00606_b200.physics import Lattice, gvector_set, l_of_lm, synthetic_system


def test_gvector_set_properties():
    lat = Lattice.cubic(10.0)
    g = gvector_set(lat, (0.0, 0.0, 0.0), 2.0)
    assert g.dtype == np.int32 and g.shape[1] == 3
    kc = g @ lat.reciprocal
    assert np.all(np.linalg.norm(kc, axis=1) <= 2.0)
    # lexicographic, unique, inversion-symmetric at Gamma
    assert np.all(np.diff(g[:, 0]) >= 0)
    assert len({tuple(x) for x in g}) == len(g)
    assert {tuple(-x) for x in g} == {tuple(x) for x in g}
    # brute-force count over a big box
    r = np.arange(-6, 7)
    n = np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3)
    assert (np.linalg.norm(n @ lat.reciprocal, axis=1) <= 2.0).sum() == len(g)
    # shifted k: set follows |k+G|
    gk = gvector_set(lat, (0.25, 0.0, -0.5), 2.0)
    assert np.all(np.linalg.norm((gk + [0.25, 0, -0.5]) @ lat.reciprocal, axis=1) <= 2.0)


@pytest.mark.parametrize("target", [500, 3000])
def test_synthetic_system_hits_target_ng(target):
    system, k, kmax, g = synthetic_system(8, 2, 8, target, seed=1)
    assert abs(len(g) - target) <= 0.01 * target
    assert system.n_l == 81 and len(system.u_norms()) == 8
    assert np.array_equal(l_of_lm(2), [0, 1, 1, 1, 2, 2, 2, 2, 2])


def test_ylm_known_answers():
    # Y_00 = 1/sqrt(4 pi); Y_10 = sqrt(3/4pi) cos(theta); Y_11 = -sqrt(3/8pi) sin(theta) e^{i phi}
    kc = np.array([[0.3, -0.4, 1.2], [0.0, 0.0, 2.0], [1.0, 1.0, 0.0]])
    y = om.ylm_all(1, kc)
    kn = np.linalg.norm(kc, axis=1)
    th = np.arccos(kc[:, 2] / kn)
    ph = np.arctan2(kc[:, 1], kc[:, 0])
    np.testing.assert_allclose(y[0], 1 / math.sqrt(4 * math.pi), rtol=1e-15)
    np.testing.assert_allclose(y[2], math.sqrt(3 / (4 * math.pi)) * np.cos(th), atol=1e-15)
    np.testing.assert_allclose(y[3], -math.sqrt(3 / (8 * math.pi)) * np.sin(th) * np.exp(1j * ph), atol=1e-15)
    np.testing.assert_allclose(y[1], math.sqrt(3 / (8 * math.pi)) * np.sin(th) * np.exp(-1j * ph), atol=1e-15)


def test_bessel_known_answers():
    assert sp.spherical_jn(0, 0.0) == 1.0 and sp.spherical_jn(3, 0.0) == 0.0
    x = 2.7
    assert abs(sp.spherical_jn(0, x) - math.sin(x) / x) < 1e-15
    assert abs(sp.spherical_jn(1, x) - (math.sin(x) / x**2 - math.cos(x) / x)) < 1e-15


def _one_atom(lmax=2, g=((0, 0, 0), (1, 0, 0), (0, 2, -1))):
    lat = np.eye(3) * 8.0
    radial = np.array([[[1.0, 0.3, 0.2, 1.1]] * (lmax + 1)])
    return lat, np.array([[0.5, 1.0, 2.0]]), np.array([0]), np.array([2.2]), radial, lmax, np.array(g, dtype=np.int32)


def test_gamma_column_only_l0_survives():
    lat, tau, types, rmt, radial, lmax, g = _one_atom()
    a, b = om.matching_coeffs(lat, tau, types, rmt, radial, lmax, (0, 0, 0), g)
    # column 0 is K = 0: j_l(0) = delta_l0, j_l'(0) = delta_l1 / 3, Y_00 = 1/sqrt(4pi)
    u, du, ud, dud = radial[0, 0]
    d = u * dud - ud * du
    pre = 4 * math.pi / math.sqrt(512.0)
    np.testing.assert_allclose(a[0, 0], pre / math.sqrt(4 * math.pi) * dud / d, rtol=1e-15)
    np.testing.assert_allclose(b[0, 0], pre / math.sqrt(4 * math.pi) * (-du) / d, rtol=1e-15)
    assert np.all(a[1:, 0] == 0) and np.all(b[1:, 0] == 0)


def test_single_atom_l0_closed_form():
    lat, tau, types, rmt, radial, lmax, g = _one_atom(lmax=0)
    a, b = om.matching_coeffs(lat, tau, types, rmt, radial, lmax, (0.1, 0, 0), g)
    u, du, ud, dud = radial[0, 0]
    d = u * dud - ud * du
    kc = (g + [0.1, 0, 0]) @ (2 * math.pi * np.linalg.inv(lat).T)
    for col in range(len(g)):
        K = np.linalg.norm(kc[col])
        x = K * rmt[0]
        j0, dj0 = math.sin(x) / x, (x * math.cos(x) - math.sin(x)) / x**2
        c = 4 * math.pi / math.sqrt(512.0) / math.sqrt(4 * math.pi) * np.exp(1j * kc[col] @ tau[0])
        assert abs(a[0, col] - c * (j0 * dud - K * dj0 * ud) / d) < 1e-14
        assert abs(b[0, col] - c * (K * dj0 * u - j0 * du) / d) < 1e-14
