"""Host-side description of the INT8 tensor-core engine (csrc/ozaki.cuh).

The engine emulates the FP64 complex contractions C = sum_s L_s^H R_s by the
Chinese-remainder (Ozaki-II) scheme: operands are rounded per column to
``b``-bit Gaussian integers, their residues modulo ``n_mod`` pairwise-coprime
odd moduli p_i < 256 whose prime factors are all 1 (mod 4) are split by the
isomorphism Z_p[i] = Z_p x Z_p (x + iy -> x +- j y, j^2 = -1 mod p), so each
modulus costs 2 exact real products on the INT8 tensor cores, and the
integers are reconstructed by the CRT.

``int8_moduli`` restates the library's choice (hsb_api.cu ``run_ozaki``) so
reports can count the work; the library is the authority.
"""

from __future__ import annotations

import math

MODULI = (241, 233, 229, 221, 205, 197, 193, 181, 173, 157, 149, 137, 113, 109, 101, 97)
# a square root of -1 modulo each modulus (csrc/ozaki.cuh oz_sqrtm1)
SQRT_M1 = (64, 89, 107, 21, 32, 14, 81, 19, 80, 28, 44, 37, 15, 33, 10, 22)
PRODUCTS = 2
DEFAULT_BITS = 39


def int8_moduli(k_total: int, min_bits: int = 0) -> tuple[int, int]:
    """(n_mod, b): the fewest moduli (>= 11) such that the integer bits
    b = floor((log2 M - 2 - log2 K) / 2) reach ``min_bits``: with
    |x'| + |y'| <= 2^b per element, |Re'| and |Im'| are <= K 2^(2b), which must
    stay below M / 2 (one bit of margin kept)."""
    want = min_bits or DEFAULT_BITS
    log2m = 0.0
    for i, p in enumerate(MODULI):
        log2m += math.log2(p)
        b = math.floor((log2m - 2.0 - math.log2(max(k_total, 1))) / 2.0)
        if i + 1 >= 11 and (b >= want or i + 1 == len(MODULI)):
            return i + 1, min(b, want + 4)
    raise AssertionError("unreachable")


def int8_gemm_ops(n: int, k_total: int, min_bits: int = 0) -> int:
    """Algorithmic INT8 tensor-core ops (2 per MAC) of one triangle
    contraction: 2 real products x n_mod moduli x K_tot x n(n+1)/2."""
    n_mod, _ = int8_moduli(k_total, min_bits)
    return 2 * PRODUCTS * n_mod * k_total * (n * (n + 1) // 2)
