"""Algorithm 1 on the CPU (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Restates builder.build_hs (/root/reference/pkg/src/hsgen/builder.py:211-224)
phase by phase, with the five large updates on scipy's OpenBLAS
ZHER2K/ZHERK/ZGEMM — the CPU path the paper benchmarks against
(MKL in PAPER.md:518-519):

  Loop 1  builder.py:73-88    Z_a = T_AB^H A_a + 1/2 mirror(T_BB) B_a
  H1      builder.py:91-104   lower(Z^H B + B^H Z)
  S1/U/S2 builder.py:107-132  S = A^H A + (uB)^H (uB), mirrored
  Loop 2  builder.py:162-185  potrf_lower(T_AA) -> Y = C^H A | X = mirror(T_AA) A
  H2/H3   builder.py:187-200  H += A_nh^H X_nh ; H += Y^H Y ; mirror

Returns section wall times so the bench can report the CPU baseline.
"""

from __future__ import annotations

import time

import numpy as np
import scipy.linalg.blas as blas

from .kernels import mirror, potrf_lower


def _stack(blocks):
    return np.asfortranarray(np.concatenate([np.asarray(b, dtype=np.complex128) for b in blocks], axis=0))


def _mirror_inplace(c):
    n = c.shape[0]
    iu = np.triu_indices(n, 1)
    c[iu] = np.conj(c.T[iu])
    d = np.diag_indices(n)
    c[d] = c[d].real
    return c


def build_hs_cpu(p, force_nonhpd: bool = False) -> dict:
    """H, S (full, F-order complex128), split counts and section seconds."""
    n_a, n_l, n_g = p.dims.n_atoms, p.dims.n_l, p.dims.n_g
    sec = {}
    t0 = time.perf_counter()
    a_st = _stack(p.a_blocks)
    b_st = _stack(p.b_blocks)
    z_st = np.empty_like(b_st, order="F")
    for a in range(n_a):
        r = slice(a * n_l, (a + 1) * n_l)
        z_st[r] = p.t_ab[a].conj().T @ p.a_blocks[a] + 0.5 * (mirror(p.t_bb[a]) @ p.b_blocks[a])
    t1 = time.perf_counter()
    sec["Loop 1"] = t1 - t0
    h = blas.zher2k(1.0, z_st, b_st, trans=2, lower=1)
    t2 = time.perf_counter()
    sec["H1"] = t2 - t1
    s = blas.zherk(1.0, a_st, trans=2, lower=1)
    t3 = time.perf_counter()
    sec["S1"] = t3 - t2
    u = np.concatenate([np.asarray(x, dtype=np.float64) for x in p.u_norms])
    ub = np.asfortranarray(b_st * u[:, None])
    t4 = time.perf_counter()
    sec["U norm"] = t4 - t3
    s = blas.zherk(1.0, ub, beta=1.0, c=s, trans=2, lower=1, overwrite_c=1)
    s = _mirror_inplace(np.asfortranarray(s))
    t5 = time.perf_counter()
    sec["S2"] = t5 - t4
    ys, xs, anh = [], [], []
    hpd = 0
    for a in range(n_a):
        factor = None
        if not force_nonhpd:
            factor, _ = potrf_lower(p.t_aa[a])
        if factor is not None:
            ys.append(factor.conj().T @ p.a_blocks[a])
            hpd += 1
        else:
            xs.append(mirror(p.t_aa[a]) @ p.a_blocks[a])
            anh.append(np.asarray(p.a_blocks[a]))
    t6 = time.perf_counter()
    sec["Loop 2"] = t6 - t5
    h = np.asfortranarray(h)
    if xs:
        prod = blas.zgemm(1.0, _stack(anh), _stack(xs), trans_a=2)
        h += prod  # full-matrix update, as the reference's GEMM (builder.py:188-192)
    t7 = time.perf_counter()
    sec["H2"] = t7 - t6
    if ys:
        h = blas.zherk(1.0, _stack(ys), beta=1.0, c=h, trans=2, lower=1, overwrite_c=1)
    h = _mirror_inplace(np.asfortranarray(h))
    t8 = time.perf_counter()
    sec["H3"] = t8 - t7
    return {"h": h, "s": s, "hpd": hpd, "nonhpd": n_a - hpd, "seconds": sec, "total": t8 - t0}
