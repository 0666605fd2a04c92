"""Host-side description of the INT8 tensor-core engine (csrc/ozaki.cuh).

The engine emulates the FP64 complex contractions C = sum_s L_s^H R_s by the
Chinese-remainder (Ozaki-II) scheme: operands are rounded per column to
``b``-bit integers, their residues modulo ``n_mod`` pairwise-coprime moduli
p_i <= 256 are multiplied exactly on the INT8 tensor cores (3 real products
per modulus, Gauss/3M), and the integers are reconstructed by the CRT.

``int8_moduli`` restates the library's choice (hsb_api.cu ``run_ozaki``) so
reports can count the work; the library is the authority.
"""

from __future__ import annotations

import math

MODULI = (256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193)
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
    contraction: 3 real products x n_mod moduli x K_tot x n(n+1)/2."""
    n_mod, _ = int8_moduli(k_total, min_bits)
    return 2 * 3 * n_mod * k_total * (n * (n + 1) // 2)
