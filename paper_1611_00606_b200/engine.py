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
from fractions import Fraction

MODULI = (241, 233, 229, 221, 205, 197, 193, 181, 173, 157, 149, 137, 113, 109, 101, 97, 89, 73, 61, 53)
# a square root of -1 modulo each modulus (csrc/ozaki.cuh oz_sqrtm1)
SQRT_M1 = (64, 89, 107, 21, 32, 14, 81, 19, 80, 28, 44, 37, 15, 33, 10, 22, 34, 27, 11, 23)
PRODUCTS = 2
MIN_MODULI = 11
DEFAULT_BITS = 53   # a full FP64 mantissa per operand (csrc/ozaki.cuh kOzDefaultBits)
MAX_BITS = 55       # csrc/ozaki.cuh kOzMaxBits


def int8_moduli(k_total: int, min_bits: int = 0) -> tuple[int, int]:
    """(n_mod, b): the fewest moduli (>= 11) such that the integer bits
    b = floor((log2 M - 2 - log2 K) / 2) reach ``min_bits``: with
    |x'| + |y'| <= 2^b per element, |Re'| and |Im'| are <= K 2^(2b), which must
    stay below M / 2 (one bit of margin kept).  b is then raised as far as
    those moduli allow, up to MAX_BITS (contract.cu ``oz_choose``)."""
    want = min_bits or DEFAULT_BITS
    log2m = 0.0
    for i, p in enumerate(MODULI):
        log2m += math.log2(p)
        b = math.floor((log2m - 2.0 - math.log2(max(k_total, 1))) / 2.0)
        if i + 1 >= MIN_MODULI and (b >= want or i + 1 == len(MODULI)):
            return i + 1, min(b, MAX_BITS)
    raise AssertionError("unreachable")


def int8_gemm_ops(n: int, k_total: int, min_bits: int = 0) -> int:
    """Algorithmic INT8 tensor-core ops (2 per MAC) of one triangle
    contraction: 2 real products x n_mod moduli x K_tot x n(n+1)/2."""
    n_mod, _ = int8_moduli(k_total, min_bits)
    return 2 * PRODUCTS * n_mod * k_total * (n * (n + 1) // 2)


def crt_weights(n_mod: int) -> tuple[list[list[tuple[float, float]]], float]:
    """The reconstruction tables of csrc/ozaki.cu ``oz_crt_table``: for the Re
    (c = 1/2) and Im (c = 1/(2 j)) parts, u_i / p_i with
    u_i = c (M / p_i)^-1 mod p_i as two 40-bit fixed-point limbs (rounded to
    nearest at 2^-80), and fl(M)."""
    mods = MODULI[:n_mod]
    big_m = math.prod(mods)
    out = []
    for part in range(2):
        row = []
        for i, p in enumerate(mods):
            c = pow(2, -1, p) if part == 0 else pow(2 * SQRT_M1[i], -1, p)
            u = c * pow(big_m // p % p, -1, p) % p
            q = ((u << 80) + p // 2) // p
            row.append((math.ldexp(q >> 40, -40), math.ldexp(q & ((1 << 40) - 1), -80)))
        out.append(row)
    return out, float(Fraction(big_m))


def crt_fraction(residues, weights) -> float:
    """X / M from the residues of one part (csrc/ozaki.cu ``crt_frac``):
    s1 = sum r_i w_i1 (exact), s2 = sum r_i w_i2, f = (s1 - rint(s1)) + s2."""
    s1 = s2 = 0.0
    for r, (w1, w2) in zip(residues, weights):
        s1 += float(r) * w1
        s2 += float(r) * w2
    return (s1 - float(round(s1))) + s2
