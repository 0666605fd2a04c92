"""Kernel-level parity on the B200: the DMMA contraction kernel through the
C ABI (via the run_partitioned drop-in) against the reference's own kernel
outputs (tests/golden/kernels.npz) and the CPU oracle at larger sizes.
Tolerance: relative Frobenius 1e-12 (north star requires <= 1e-10)."""

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import kernels as ok
from paper_1611_00606_b200 import (DimensionError, GpuPolicy, InputError, KernelKind, rel_frob_error,
                                   run_partitioned)

pytestmark = pytest.mark.gpu
TOL = 1e-12
TOL_INT8 = 1e-13  # the INT8 engine at FP64 width (>= 53-bit operands); the north star asks for 1e-10


def _tol(pol):
    return TOL_INT8 if pol.engine == "int8" else TOL


@pytest.fixture(scope="module")
def g():
    with np.load(GOLDEN / "kernels.npz") as z:
        return {k: z[k] for k in z.files}


def _cm(rng, r, c):
    return np.asfortranarray(rng.standard_normal((r, c)) + 1j * rng.standard_normal((r, c)))


@pytest.fixture(params=["3m", "4m", "int8"])
def pol(request):
    if request.param == "int8":  # INT8 tensor-core CRT emulation of the triangle updates
        return GpuPolicy(engine="int8")
    return GpuPolicy(engine="dmma", complex_mult=request.param)


def test_herk_matches_reference_kernel(g, pol):
    i = 0
    while f"herk{i}_a" in g:
        alpha, beta = (float(x) for x in g[f"herk{i}_ab"])
        c = g[f"herk{i}_c"].copy(order="F")
        res = run_partitioned(KernelKind.HERK, (alpha, g[f"herk{i}_a"], beta, c), pol)
        assert rel_frob_error(c, g[f"herk{i}_out"]) < _tol(pol), i
        assert res.seconds >= 0 and res.n_tiles >= 1
        i += 1


def test_her2k_matches_reference_kernel(g, pol):
    i = 0
    while f"her2k{i}_z" in g:
        alpha, beta = g[f"her2k{i}_ab"]
        c = g[f"her2k{i}_c"].copy(order="F")
        run_partitioned(KernelKind.HER2K, (complex(alpha), g[f"her2k{i}_z"], g[f"her2k{i}_b"], beta.real, c), pol)
        assert rel_frob_error(c, g[f"her2k{i}_out"]) < _tol(pol), i
        assert np.all(np.diagonal(c).imag == 0)
        i += 1


def test_gemm_all_ops_match_reference_kernel(g, pol):
    i = 0
    while f"gemm{i}_a" in g:
        opa, opb = (str(x) for x in g[f"gemm{i}_ops"])
        alpha, beta = g[f"gemm{i}_ab"]
        c = g[f"gemm{i}_c"].copy(order="F")
        run_partitioned(KernelKind.GEMM, (complex(alpha), opa, g[f"gemm{i}_a"], opb, g[f"gemm{i}_b"],
                                          complex(beta), c), pol)
        assert rel_frob_error(c, g[f"gemm{i}_out"]) < _tol(pol), (i, opa, opb)
        i += 1


@pytest.mark.parametrize("k,n", [(1, 1), (3, 64), (8, 65), (121, 127), (257, 300), (2000, 700)])
def test_herk_against_oracle_sizes(k, n, pol):
    rng = np.random.default_rng(k * 1000 + n)
    a = _cm(rng, k, n)
    c = _cm(rng, n, n)
    want = ok.herk(1.0, a, 0.5, c)
    run_partitioned(KernelKind.HERK, (1.0, a, 0.5, c), pol)
    assert rel_frob_error(c, want) < _tol(pol)


@pytest.mark.parametrize("k,n", [(5, 33), (242, 190), (1000, 513)])
def test_her2k_against_oracle_sizes(k, n, pol):
    rng = np.random.default_rng(7 + k + n)
    z, b = _cm(rng, k, n), _cm(rng, k, n)
    c = _cm(rng, n, n)
    want = ok.her2k(1.0, z, b, 0.0, c)
    run_partitioned(KernelKind.HER2K, (1.0, z, b, 0.0, c), pol)
    assert rel_frob_error(c, want) < _tol(pol)


def test_zero_alpha_and_empty_reduction_follow_blas():
    rng = np.random.default_rng(3)
    a = _cm(rng, 4, 9)
    c = _cm(rng, 9, 9)
    want = ok.herk(0.0, a, 2.0, c)
    run_partitioned(KernelKind.HERK, (0.0, a, 2.0, c))
    assert rel_frob_error(c, want) < TOL
    c2 = _cm(rng, 9, 9)
    want2 = ok.gemm(1.0, "C", np.zeros((0, 9), complex), "N", np.zeros((0, 9), complex), 0.0, c2)
    run_partitioned(KernelKind.GEMM, (1.0, "C", np.zeros((0, 9), complex), "N", np.zeros((0, 9), complex), 0.0, c2))
    assert np.array_equal(c2, want2)


def test_errors_match_reference_classes():
    rng = np.random.default_rng(4)
    a = _cm(rng, 4, 5)
    with pytest.raises(DimensionError):
        run_partitioned(KernelKind.HERK, (1.0, a, 0.0, _cm(rng, 4, 4)))
    with pytest.raises(InputError):
        run_partitioned(KernelKind.HERK, (1.0 + 1j, a, 0.0, _cm(rng, 5, 5)))
    with pytest.raises(InputError):
        run_partitioned(KernelKind.GEMM, (1.0, "X", a, "N", a, 0.0, _cm(rng, 5, 5)))
    with pytest.raises(InputError):
        run_partitioned(KernelKind.POTRF, (a,))


@pytest.mark.parametrize("k,n", [(17000, 260), (40000, 130), (9000, 513)])
def test_int8_engine_long_reductions_use_several_slabs(k, n):
    # k > 16384 bytes of reduction: the INT8 GEMM splits k into slabs whose
    # residues are summed in the CRT (C4's H call has three)
    rng = np.random.default_rng(k + n)
    z, b = _cm(rng, k, n), _cm(rng, k, n)
    c = _cm(rng, n, n)
    want = ok.her2k(1.0, z, b, 0.0, c)
    run_partitioned(KernelKind.HER2K, (1.0, z, b, 0.0, c), GpuPolicy(engine="int8"))
    assert rel_frob_error(c, want) < TOL_INT8
    a = _cm(rng, k, n)
    c2 = _cm(rng, n, n)
    want2 = ok.herk(0.5, a, 2.0, c2)
    run_partitioned(KernelKind.HERK, (0.5, a, 2.0, c2), GpuPolicy(engine="int8"))
    assert rel_frob_error(c2, want2) < TOL_INT8


def test_int8_engine_is_column_scale_invariant():
    # the INT8 engine scales every column to its own exponent, so columns whose
    # magnitudes differ by 300 orders (and an all-zero column) keep ~2^-40
    # accuracy relative to sqrt(C_mm C_nn) element by element
    rng = np.random.default_rng(5)
    k, n = 700, 300
    a = _cm(rng, k, n)
    scale = 10.0 ** rng.uniform(-150, 150, n)
    a *= scale[None, :]
    a[:, 7] = 0
    c = np.zeros((n, n), complex, order="F")
    want = ok.herk(1.0, a, 0.0, c.copy(order="F"))
    run_partitioned(KernelKind.HERK, (1.0, a, 0.0, c), GpuPolicy(engine="int8"))
    want = np.tril(want)
    got = np.tril(c)
    d = np.sqrt(np.abs(np.diag(want)))
    norm = np.outer(d, d)
    norm[norm == 0] = 1.0
    assert np.all(got[:, 7] == 0) and np.all(got[7, :] == 0)
    assert np.max(np.abs(got - want) / norm) < 1e-10


@pytest.mark.parametrize("engine", ["int8", "dmma"])
@pytest.mark.parametrize("opa", ["C", "T"])
def test_gemmt_lower_only_through_the_abi(engine, opa):
    # hsb_zgemm with HSB_LOWER_ONLY (GEMMT): a triangle call; with opa 'T' the
    # INT8 engine takes its non-conjugating path (Re = P - Q, Im = W - P - Q)
    import ctypes

    import torch

    from paper_1611_00606_b200 import _lib

    rng = np.random.default_rng(11)
    k, n = 333, 290
    a, b = _cm(rng, k, n), _cm(rng, k, n)
    c0 = _cm(rng, n, n)
    dev = torch.device("cuda", 0)
    da = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)   # row-major (n, k) = column-major k x n
    db = torch.from_numpy(np.ascontiguousarray(b.T)).to(dev)
    dc = torch.from_numpy(np.ascontiguousarray(c0.T)).to(dev)
    lib = _lib.load()
    ctx = _lib.context(0, "3m", engine)
    st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(lib.hsb_zgemm(ctx, st, opa.encode(), b"N", n, n, k, 1.0, 0.0, da.data_ptr(), k, db.data_ptr(), k,
                             0.5, 0.0, dc.data_ptr(), n, _lib.HSB_LOWER_ONLY), ctx)
    torch.cuda.synchronize()
    got = dc.cpu().numpy().T
    opm = a.conj().T if opa == "C" else a.T
    want = opm @ b + 0.5 * c0
    low = np.tril_indices(n)
    err = np.linalg.norm(got[low] - want[low]) / (1 + np.linalg.norm(want[low]))
    assert err < (TOL_INT8 if engine == "int8" else TOL)
    up = np.triu_indices(n, 1)
    assert np.array_equal(got[up], c0[up])  # the strict upper triangle is untouched
    _lib.context(0, "3m", "int8")  # restore the default engine for later tests
