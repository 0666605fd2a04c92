"""Matching coefficients on the CPU (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

PARITY UNPINNED BY THE REFERENCE: the reference has no implementation of
this row (A and B are random inputs there, probgen.py:131-132; SPEC.md:323
treats L as a flat index).  This restatement follows the paper's
definition with the conventions fixed in SURVEY.md 8(a)
row A0, and is pinned instead by closed forms (tests/test_matching_cpu.py:
Y_00, Y_1m, j_l(0), the Gamma-point column, a single-atom l = 0 case) and by
scipy's special functions, which are an implementation independent of the
GPU kernel's recurrences:

    Y_lm   scipy.special.sph_harm_y(l, m, theta, phi)  (Condon-Shortley phase)
    j_l    scipy.special.spherical_jn(l, x[, derivative=True])

    c_lm = (4 pi / sqrt(Omega)) i^l exp(i K.tau) conj(Y_lm(K^))
    A    = c [ j_l udot' - K j_l' udot ] / D,   B = c [ K j_l' u - j_l u' ] / D
"""

from __future__ import annotations

import math

import numpy as np
import scipy.special as sp


def lm_pairs(lmax: int):
    return [(l, m) for l in range(lmax + 1) for m in range(-l, l + 1)]


def kvectors(lattice_vectors, kpt_frac, gset):
    b = 2.0 * math.pi * np.linalg.inv(np.asarray(lattice_vectors, dtype=np.float64)).T
    return (np.asarray(gset, dtype=np.float64) + np.asarray(kpt_frac, dtype=np.float64)) @ b


def ylm_all(lmax: int, kc: np.ndarray) -> np.ndarray:
    """(N_L, n_g) complex Y_lm(K^); direction of K = 0 taken as theta = phi = 0."""
    kn = np.linalg.norm(kc, axis=1)
    safe = np.where(kn > 0, kn, 1.0)
    cost = np.where(kn > 0, kc[:, 2] / safe, 1.0)
    theta = np.arccos(np.clip(cost, -1.0, 1.0))
    phi = np.mod(np.arctan2(kc[:, 1], kc[:, 0]), 2 * math.pi)
    phi = np.where(kn > 0, phi, 0.0)
    return np.stack([sp.sph_harm_y(l, m, theta, phi) for l, m in lm_pairs(lmax)])


def matching_coeffs(lattice_vectors, positions, types, rmt, radial, lmax, kpt_frac, gset):
    """Stacked A, B (K x n_g, column-major complex128), rows (atom, L) atom-major."""
    kc = kvectors(lattice_vectors, kpt_frac, gset)
    kn = np.linalg.norm(kc, axis=1)
    omega = abs(np.linalg.det(np.asarray(lattice_vectors, dtype=np.float64)))
    pre = 4.0 * math.pi / math.sqrt(omega)
    ls = np.array([l for l, _ in lm_pairs(lmax)])
    yconj = np.conj(ylm_all(lmax, kc)) * (1j ** ls)[:, None] * pre          # (N_L, n_g)
    n_a, n_l = len(types), len(ls)
    a_st = np.empty((n_a * n_l, kc.shape[0]), dtype=np.complex128, order="F")
    b_st = np.empty_like(a_st, order="F")
    radial = np.asarray(radial, dtype=np.float64)
    for al in range(n_a):
        t = int(types[al])
        x = kn * rmt[t]
        phase = np.exp(1j * (kc @ np.asarray(positions[al], dtype=np.float64)))
        for l in range(lmax + 1):
            u, du, ud, dud = radial[t, l]
            d = u * dud - ud * du
            jl = sp.spherical_jn(l, x)
            djl = sp.spherical_jn(l, x, derivative=True)
            fa = (jl * dud - kn * djl * ud) / d
            fb = (kn * djl * u - jl * du) / d
            rows = slice(al * n_l + l * l, al * n_l + (l + 1) ** 2)
            base = yconj[l * l:(l + 1) ** 2] * phase[None, :]
            a_st[rows] = base * fa[None, :]
            b_st[rows] = base * fb[None, :]
    return a_st, b_st
