"""Pin the CPU oracle against fixtures produced by the reference itself.

Fixtures: tests/golden/make_golden.py ran hsgen.build_hs, hsgen.reference and
hsgen.kernels (/root/reference/pkg/src/hsgen) on seeded instances.  The
oracle must reproduce them before it may judge the GPU path.
"""

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, load_case
from oracle import alg1, brute
from oracle import kernels as ok
from paper_1611_00606_b200 import rel_frob_error


def _digest(p):
    h = hashlib.sha256()
    for name in ("a_blocks", "b_blocks", "t_aa", "t_ab", "t_bb", "u_norms"):
        for blk in getattr(p, name):
            h.update(np.asarray(blk).tobytes(order="F"))
    return h.hexdigest()


@pytest.mark.parametrize("name", golden_cases())
def test_generator_port_is_bit_identical(name):
    # probgen.generate (probgen.py:119-137) restated in instances.generate
    p, _, meta = load_case(name)
    assert _digest(p) == meta["digest"]


@pytest.mark.parametrize("name", golden_cases())
def test_alg1_oracle_matches_reference_build(name):
    p, fx, meta = load_case(name)
    out = alg1.build_hs_cpu(p, force_nonhpd=meta["force_nonhpd"])
    assert [out["hpd"], out["nonhpd"]] == fx["split"].tolist()
    assert rel_frob_error(out["h"], fx["h"]) < 1e-13
    assert rel_frob_error(out["s"], fx["s"]) < 1e-13


@pytest.mark.parametrize("name", [n for n in golden_cases() if n != "c1"])
def test_brute_oracle_matches_reference_oracle(name):
    p, fx, _ = load_case(name)
    assert rel_frob_error(brute.h_brute(p), fx["h_ref"]) < 1e-13
    assert rel_frob_error(brute.s_brute(p), fx["s_ref"]) < 1e-13
    # and the reference's own build agrees with its oracle (acceptance crit. 3)
    assert rel_frob_error(fx["h"], fx["h_ref"]) < 1e-12


def test_kernel_oracles_match_reference_kernels():
    with np.load(GOLDEN / "kernels.npz") as z:
        g = {k: z[k] for k in z.files}
    i = 0
    while f"herk{i}_a" in g:
        alpha, beta = g[f"herk{i}_ab"]
        got = ok.herk(alpha, g[f"herk{i}_a"], beta, g[f"herk{i}_c"])
        assert rel_frob_error(got, g[f"herk{i}_out"]) < 1e-14, i
        i += 1
    i = 0
    while f"her2k{i}_z" in g:
        alpha, beta = g[f"her2k{i}_ab"]
        got = ok.her2k(alpha, g[f"her2k{i}_z"], g[f"her2k{i}_b"], beta.real, g[f"her2k{i}_c"])
        assert rel_frob_error(got, g[f"her2k{i}_out"]) < 1e-14, i
        i += 1
    i = 0
    while f"gemm{i}_a" in g:
        opa, opb = (str(x) for x in g[f"gemm{i}_ops"])
        alpha, beta = g[f"gemm{i}_ab"]
        got = ok.gemm(alpha, opa, g[f"gemm{i}_a"], opb, g[f"gemm{i}_b"], beta, g[f"gemm{i}_c"])
        assert rel_frob_error(got, g[f"gemm{i}_out"]) < 1e-14, i
        i += 1
    i = 0
    while f"potrf{i}_t" in g:
        f, info = ok.potrf_lower(g[f"potrf{i}_t"])
        assert info == int(g[f"potrf{i}_info"]) == 0
        assert rel_frob_error(f, g[f"potrf{i}_f"]) < 1e-14
        f2, info2 = ok.potrf_lower(g[f"potrf{i}_t_bad"])
        assert f2 is None and info2 == int(g[f"potrf{i}_info_bad"])
        i += 1


def test_potrf_known_answers():
    # pkg/tests/test_kernels.py:237-255
    f, info = ok.potrf_lower(np.eye(3, dtype=complex))
    assert info == 0 and np.array_equal(f, np.eye(3))
    f, info = ok.potrf_lower(np.array([[4.0]], dtype=complex))
    assert info == 0 and f[0, 0] == 2.0
    f, info = ok.potrf_lower(np.array([[1, 0], [2, 1]], dtype=complex))
    assert f is None and info == 2
