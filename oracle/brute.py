"""Defining sums of H and S (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Restates reference.s_reference / h_reference
(/root/reference/pkg/src/hsgen/reference.py:22-91; Eqs. 4-7):

  S = sum_a A_a^H A_a + (U_a B_a)^H (U_a B_a)
  H = sum_a A^H T_AA A + A^H T_AB B + B^H T_AB^H A + B^H T_BB B

with T_AA, T_BB taken as hermitian_mirror of their lower triangles (the
builder's convention, kernels.py:223-231).  No half-trick, no Cholesky,
no stacking: an independent cross-check of the Algorithm-1 restatement,
vectorised per atom (numpy matmul) instead of the reference's scalar loops.
"""

from __future__ import annotations

import numpy as np

from .kernels import mirror


def s_brute(p) -> np.ndarray:
    n_g = p.dims.n_g
    s = np.zeros((n_g, n_g), dtype=np.complex128)
    for a in range(p.dims.n_atoms):
        A = np.asarray(p.a_blocks[a])
        UB = np.asarray(p.u_norms[a])[:, None] * np.asarray(p.b_blocks[a])
        s += A.conj().T @ A + UB.conj().T @ UB
    return np.asfortranarray(s)


def h_brute(p) -> np.ndarray:
    n_g = p.dims.n_g
    h = np.zeros((n_g, n_g), dtype=np.complex128)
    for a in range(p.dims.n_atoms):
        A, B = np.asarray(p.a_blocks[a]), np.asarray(p.b_blocks[a])
        taa, tab, tbb = mirror(p.t_aa[a]), np.asarray(p.t_ab[a]), mirror(p.t_bb[a])
        h += A.conj().T @ (taa @ A) + A.conj().T @ (tab @ B)
        h += B.conj().T @ (tab.conj().T @ A) + B.conj().T @ (tbb @ B)
    return np.asfortranarray(h)
