"""Kernel-level CPU restatements (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Each function restates one serial kernel of the reference
(/root/reference/pkg/src/hsgen/kernels.py) with numpy arithmetic instead of
the reference's ascending-k rank-1 loop; results agree to rounding, which is
what the 1e-10 parity bar (north star) needs.
"""

from __future__ import annotations

import math

import numpy as np


def mirror(t: np.ndarray) -> np.ndarray:
    """matcore.hermitian_mirror (matcore.py:89-105): lower -> full, real diagonal."""
    low = np.tril(t, -1)
    return low + low.conj().T + np.diag(np.diagonal(t).real)


def _op(op, m):
    return {"N": m, "T": m.T, "C": m.conj().T}[op]


def _tail_lower(c, prod, beta):
    """kernels._update_lower (kernels.py:234-253)."""
    c = np.array(c, dtype=np.complex128, order="F")
    il = np.tril_indices(c.shape[0])
    if prod is None:
        new = 0 * c[il] if beta == 0 else beta * c[il]
    else:
        new = prod[il] if beta == 0 else prod[il] + beta * c[il]
    c[il] = new
    d = np.diag_indices(c.shape[0])
    c[d] = c[d].real
    return c


def herk(alpha, a, beta, c):
    """kernels.herk (kernels.py:256-264): lower(alpha a^H a + beta c)."""
    prod = None if alpha == 0 else alpha * (a.conj().T @ a)
    return _tail_lower(c, prod, beta)


def her2k(alpha, z, b, beta, c):
    """kernels.her2k (kernels.py:267-281): lower(alpha z^H b + conj(alpha) b^H z + beta c)."""
    prod = None if alpha == 0 else alpha * (z.conj().T @ b) + np.conj(alpha) * (b.conj().T @ z)
    return _tail_lower(c, prod, beta)


def gemm(alpha, opa, a, opb, b, beta, c):
    """kernels.gemm (kernels.py:195-220): alpha op(a) op(b) + beta c (full)."""
    prod = None if alpha == 0 else alpha * (_op(opa, a) @ _op(opb, b))
    if prod is None:
        return np.zeros_like(c) if beta == 0 else beta * c
    return prod if beta == 0 else prod + beta * c


def potrf_lower(t):
    """kernels.potrf_lower (kernels.py:296-325), same left-looking order.

    Returns (factor, 0) on success or (None, k) with k the 1-based order of the
    first non-positive leading minor.
    """
    n = t.shape[0]
    f = np.zeros((n, n), dtype=np.complex128)
    for j in range(n):
        row = f[j, :j]
        d = float(t[j, j].real) - float(np.sum(row.real * row.real + row.imag * row.imag))
        if not d > 0.0:
            return None, j + 1
        ljj = math.sqrt(d)
        f[j, j] = ljj
        if j + 1 < n:
            col = np.array(t[j + 1:, j], dtype=np.complex128) - f[j + 1:, :j] @ np.conj(row)
            f[j + 1:, j] = col / ljj
    return f, 0
