"""Pipeline-level parity on the B200: build_hs (the drop-in for
hsgen.builder.build_hs) against the reference's own outputs
(tests/golden/, produced by running hsgen) and against the CPU oracle.
Tolerance: relative Frobenius 1e-10 on H and S (north star)."""

import numpy as np
import pytest

from conftest import golden_cases, load_case
from oracle import alg1, brute
from paper_1611_00606_b200 import (
    CONFIGS, DeviceProblem, Dims, Fill, GpuPolicy, InvariantError, ProblemInstance, ProblemSpec, build_hs,
    build_hs_device, generate, rel_frob_error, section_flops,
)

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _pol(cm, **kw):
    """complex-product form "3m" / "4m" on DMMA, or the INT8 CRT engine"""
    return GpuPolicy(engine="int8", **kw) if cm == "int8" else GpuPolicy(engine="dmma", complex_mult=cm, **kw)


@pytest.mark.parametrize("cm", ["3m", "4m", "int8"])
@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("name", golden_cases())
def test_build_matches_reference_golden(name, fused, cm):
    p, fx, meta = load_case(name)
    out = build_hs(p, _pol(cm, fused=fused), force_nonhpd=meta["force_nonhpd"])
    assert [out.split.hpd, out.split.nonhpd] == fx["split"].tolist()
    assert rel_frob_error(out.h.matrix, fx["h"]) < TOL
    assert rel_frob_error(out.s.matrix, fx["s"]) < TOL
    if "h_ref" in fx:  # the reference's brute-force oracle
        assert rel_frob_error(out.h.matrix, fx["h_ref"]) < TOL
        assert rel_frob_error(out.s.matrix, fx["s_ref"]) < TOL
    assert out.h.fill is Fill.FULL and out.s.fill is Fill.FULL
    out.h.check()
    out.s.check()
    assert [r.kind.value for r in out.ledger] == [str(k) for k in fx["ledger_kind"]]
    assert [r.section for r in out.ledger] == [str(s) for s in fx["ledger_section"]]
    assert out.ledger.total_flops() == int(fx["ledger_flops"].sum())


def _scalar_instance(a, b, t, u, v, w):
    inst = ProblemInstance(Dims(1, 1, 1))
    inst.a_blocks.append(np.array([[a]], dtype=complex, order="F"))
    inst.b_blocks.append(np.array([[b]], dtype=complex, order="F"))
    inst.t_aa.append(np.array([[t]], dtype=complex, order="F"))
    inst.t_ab.append(np.array([[u]], dtype=complex, order="F"))
    inst.t_bb.append(np.array([[v]], dtype=complex, order="F"))
    inst.u_norms.append(np.array([w], dtype=float))
    return inst


@pytest.mark.parametrize("cm,rtol", [("3m", 1e-14), ("4m", 1e-14), ("int8", 1e-14)])
def test_scalar_closed_form(cm, rtol):
    # pkg/tests/test_builder.py:242-248: H = t + 2 Re(u) + v, S = 1 + w^2, at the
    # reference's own tolerance on every engine (the INT8 engine keeps >= 53
    # bits of each column's max)
    t, v, w, u = 0.7, 1.3, 0.6, 0.2 - 0.4j
    out = build_hs(_scalar_instance(1.0, 1.0, t, u, v, w), _pol(cm))
    np.testing.assert_allclose(out.h.matrix, [[t + 2 * u.real + v]], rtol=rtol)
    np.testing.assert_allclose(out.s.matrix, [[1 + w**2]], rtol=rtol)


@pytest.mark.parametrize("dims,frac", [((1, 2, 4), 0.0), ((6, 12, 48), 0.5), ((3, 81, 200), 1.0),
                                       ((2, 130, 70), 0.5), ((9, 16, 1), 0.0)])
@pytest.mark.parametrize("cm", ["3m", "4m", "int8"])
def test_build_sweep_against_brute_oracle(dims, frac, cm):
    p = generate(ProblemSpec(Dims(*dims), seed=sum(dims), nonhpd_fraction=frac))
    out = build_hs(p, _pol(cm))
    assert rel_frob_error(out.h.matrix, brute.h_brute(p)) < TOL
    assert rel_frob_error(out.s.matrix, brute.s_brute(p)) < TOL
    assert out.split.hpd + out.split.nonhpd == dims[0]


def test_c2_against_alg1_oracle():
    p = generate(ProblemSpec(CONFIGS["C2"], seed=0, nonhpd_fraction=0.25))
    out = build_hs(p)
    ref = alg1.build_hs_cpu(p)
    assert (out.split.hpd, out.split.nonhpd) == (ref["hpd"], ref["nonhpd"])
    assert rel_frob_error(out.h.matrix, ref["h"]) < TOL
    assert rel_frob_error(out.s.matrix, ref["s"]) < TOL
    tot = out.ledger.section_totals()
    assert {k: v[0] for k, v in tot.items()} == {k: v for k, v in section_flops(p.dims, ref["nonhpd"]).items() if v}


def test_forced_branch_matches_cholesky_path():
    # acceptance criterion 4 (pkg/tests/test_acceptance.py:72-87)
    p = generate(ProblemSpec(Dims(4, 24, 150), seed=1000, nonhpd_fraction=0.0))
    normal = build_hs(p)
    forced = build_hs(p, force_nonhpd=True)
    assert normal.split.nonhpd == 0 and forced.split.hpd == 0
    assert rel_frob_error(forced.h.matrix, normal.h.matrix) < 1e-10
    assert "H2" in forced.ledger.section_totals() and "H3" not in forced.ledger.section_totals()


def test_restore_contract_and_determinism():
    p = generate(ProblemSpec(Dims(3, 20, 140), seed=17, nonhpd_fraction=0.5))
    before = [m.tobytes() for m in (*p.a_blocks, *p.b_blocks)]
    o1 = build_hs(p)
    o2 = build_hs(p)
    assert [m.tobytes() for m in (*p.a_blocks, *p.b_blocks)] == before
    # same kernels, same schedule: bitwise reproducible (cf. criterion 5)
    assert o1.h.matrix.tobytes() == o2.h.matrix.tobytes()
    assert o1.s.matrix.tobytes() == o2.s.matrix.tobytes()


def test_rejects_invalid_instance_before_work():
    p = generate(ProblemSpec(Dims(2, 3, 4), seed=20))
    p.t_aa[0][0, 1] += 1.0
    with pytest.raises(InvariantError):
        build_hs(p)


def _corrupt(p, edits):
    for field, atom, idx, value in edits:
        blk = getattr(p, field)[atom]
        if idx == "shape":
            getattr(p, field)[atom] = blk[:-1]
        else:
            blk[idx] = value
    return p


@pytest.mark.parametrize("edits", [
    [("t_aa", 1, (0, 2), 1.0 + 0.5j)],                          # off-diagonal defect
    [("t_bb", 2, (3, 3), 1.0 + 1e-9j)],                         # imaginary diagonal
    [("t_ab", 0, (1, 1), np.nan)],
    [("u_norms", 1, 2, -1.0)],
    [("u_norms", 2, 0, np.inf)],
    [("t_bb", 0, (0, 1), 2.0), ("t_aa", 2, (1, 1), np.inf)],     # finiteness before Hermitian
    [("t_bb", 1, (2, 2), np.nan), ("t_ab", 2, (0, 0), np.nan)],  # field order
    [("t_aa", 2, (0, 1), 3.0), ("t_aa", 1, (0, 1), 3.0)],        # atom order
    [("u_norms", 0, 0, -1.0), ("t_bb", 2, (0, 1), 3.0)],        # Hermitian before u > 0
    [("t_bb", 1, "shape", None), ("t_aa", 2, (0, 0), np.nan)],   # shape after an earlier value error
    [("t_aa", 1, "shape", None), ("t_bb", 0, (0, 0), np.nan)],
])
def test_native_value_checks_follow_reference_order(edits):
    # HSB_OPT_VALIDATE checks T / u natively; the message and the precedence
    # must be those of validate_instance (probgen.py:140-168)
    from paper_1611_00606_b200 import validate_instance

    p = _corrupt(generate(ProblemSpec(Dims(3, 6, 20), seed=21)), edits)
    with pytest.raises(InvariantError) as ref:
        validate_instance(p)
    with pytest.raises(InvariantError) as got:
        build_hs(p)
    assert str(got.value) == str(ref.value)


def test_native_value_checks_accept_roundoff_hermitian():
    p = generate(ProblemSpec(Dims(3, 6, 20), seed=22))
    p.t_aa[1][0, 2] += 1e-16  # below 1e-14 (1 + ||T||_F)
    out = build_hs(p)
    assert rel_frob_error(out.s.matrix, brute.s_brute(p)) < TOL


def test_psd_and_hermitian():
    # acceptance criterion 6 (pkg/tests/test_acceptance.py:119-133)
    for seed, frac in ((0, 0.0), (1, 0.5), (2, 1.0)):
        out = build_hs(generate(ProblemSpec(Dims(4, 8, 64), seed=seed, nonhpd_fraction=frac)))
        out.h.check()
        out.s.check()
        s = out.s.matrix
        assert np.linalg.eigvalsh(s)[0] >= -1e-10 * np.linalg.norm(s)


@pytest.mark.parametrize("cm,tol", [("3m", 1e-14), ("int8", TOL)])
def test_device_path_matches_host_path(cm, tol):
    # the host path splits S into (UB)^H(UB) and A^H A launches to overlap A's
    # upload; on the INT8 engine each launch scales its own operands, so the
    # two paths agree to the engine's accuracy rather than bitwise
    import torch

    p = generate(ProblemSpec(Dims(5, 49, 333), seed=4, nonhpd_fraction=0.4))
    host = build_hs(p, _pol(cm))
    dp = DeviceProblem.from_instance(p)
    h, s, split, t, info = build_hs_device(dp, policy=_pol(cm))
    torch.cuda.synchronize()
    hm = h.cpu().numpy().T
    sm = s.cpu().numpy().T
    assert (split.hpd, split.nonhpd) == (host.split.hpd, host.split.nonhpd)
    assert rel_frob_error(hm, host.h.matrix) < tol
    assert rel_frob_error(sm, host.s.matrix) < tol
    assert t["launches"] >= 5


@pytest.mark.parametrize("field", ["a_blocks", "b_blocks"])
def test_nonfinite_stack_values_raise_invariant_error(field):
    # probgen.validate_instance (probgen.py:155-161); checked during staging
    p = generate(ProblemSpec(Dims(3, 5, 40), seed=2))
    getattr(p, field)[2][1, 7] = np.inf if field == "a_blocks" else np.nan
    with pytest.raises(InvariantError, match=rf"{field}\[2\]"):
        build_hs(p)
    # the context stays usable afterwards
    q = generate(ProblemSpec(Dims(3, 5, 40), seed=2))
    out = build_hs(q)
    assert rel_frob_error(out.s.matrix, brute.s_brute(q)) < TOL


@pytest.mark.parametrize("upper", ["", "0", "0.5", "1"])
@pytest.mark.parametrize("dims", [Dims(3, 17, 700), Dims(6, 25, 1283)])
def test_lower_triangle_download_matches_full_download(dims, upper, monkeypatch):
    # default pinned INT8 path: H / S cross PCIe as lower triangles plus a
    # fraction of the upper ones (HSB_D2H_UPPER; "" = the default split) and
    # host threads fill the rest of the upper triangles; bitwise the same as
    # full downloads
    monkeypatch.setenv("HSB_D2H_UPPER", upper)
    p = generate(ProblemSpec(dims, seed=31, nonhpd_fraction=0.3))
    a = build_hs(p, GpuPolicy(lower_d2h=True))
    b = build_hs(p, GpuPolicy(lower_d2h=False))
    c = build_hs(p, GpuPolicy(pinned_outputs=False))
    for x in (a, c):
        assert x.h.matrix.tobytes() == b.h.matrix.tobytes()
        assert x.s.matrix.tobytes() == b.s.matrix.tobytes()
    a.h.check()
    a.s.check()
    assert rel_frob_error(a.h.matrix, brute.h_brute(p)) < TOL


def test_pageable_outputs_path():
    p = generate(ProblemSpec(Dims(2, 9, 77), seed=8, nonhpd_fraction=0.5))
    a = build_hs(p, GpuPolicy(pinned_outputs=False))
    b = build_hs(p, GpuPolicy(pinned_outputs=True))
    assert a.h.matrix.tobytes() == b.h.matrix.tobytes()
    assert a.s.matrix.tobytes() == b.s.matrix.tobytes()


def test_pinned_instance_path_matches_and_checks_values():
    from paper_1611_00606_b200 import pin_instance

    p = generate(ProblemSpec(Dims(4, 33, 210), seed=12, nonhpd_fraction=0.5))
    q = pin_instance(p)
    a, b = build_hs(p), build_hs(q)
    assert rel_frob_error(b.h.matrix, a.h.matrix) < 1e-15
    assert rel_frob_error(b.s.matrix, a.s.matrix) < 1e-15
    assert rel_frob_error(b.h.matrix, brute.h_brute(p)) < TOL
    q.b_blocks[3][4, 5] = np.nan
    with pytest.raises(InvariantError, match=r"b_blocks\[3\]"):
        build_hs(q)
    q.b_blocks[3][4, 5] = 0
    q.a_blocks[1][0, 0] = -np.inf
    with pytest.raises(InvariantError, match=r"a_blocks\[1\]"):
        build_hs(q)


@pytest.mark.parametrize("cm,depth", [("3m", 2), ("int8", 2), ("int8", 3)])
def test_kpoint_pipeline_matches_serial_builds(cm, depth):
    # BASELINE config C5 on one GPU: independent k-points through several
    # contexts and streams, chained by upload / compute events; each result
    # equals its serial build bitwise (k-points of different sizes included)
    from paper_1611_00606_b200 import build_hs_kpoints

    ps = [generate(ProblemSpec(Dims(3, 25, 260 + 37 * (i % 3)), seed=40 + i, nonhpd_fraction=0.3))
          for i in range(7)]
    serial = [build_hs(p, _pol(cm)) for p in ps]
    piped = build_hs_kpoints(ps, _pol(cm), depth=depth)
    for a, b, p in zip(serial, piped, ps):
        assert a.h.matrix.tobytes() == b.h.matrix.tobytes()
        assert a.s.matrix.tobytes() == b.s.matrix.tobytes()
        assert (a.split.hpd, a.split.nonhpd) == (b.split.hpd, b.split.nonhpd)
        assert rel_frob_error(b.h.matrix, brute.h_brute(p)) < TOL


@pytest.mark.timeout(120)
def test_kpoint_iterator_early_exit_and_slow_consumer():
    # the window flow control must neither deadlock when a lane runs ahead
    # (staggered start) nor leave lanes blocked when the consumer stops early
    import time

    from paper_1611_00606_b200 import iter_hs_kpoints

    ps = [generate(ProblemSpec(Dims(2, 16, 120), seed=90 + i)) for i in range(7)]
    got = []
    for i, out in enumerate(iter_hs_kpoints(ps, _pol("int8"), depth=2)):
        time.sleep(0.02)  # slow consumer
        got.append(out.split.hpd + out.split.nonhpd)
        if i == 3:
            break  # generator closed with lanes still running
    assert got == [2, 2, 2, 2]
    assert len(list(iter_hs_kpoints(ps, _pol("int8"), depth=3))) == 7


@pytest.mark.timeout(120)
def test_kpoint_pipeline_failure_mid_batch_does_not_hang():
    # a k-point that fails validation on the device (non-finite A) must surface
    # as the reference's InvariantError without leaving later k-points waiting
    # on its upload / compute events
    from paper_1611_00606_b200 import iter_hs_kpoints

    from paper_1611_00606_b200 import pin_instance

    ps = [pin_instance(generate(ProblemSpec(Dims(2, 16, 140), seed=120 + i))) for i in range(6)]
    ps[2].a_blocks[1][3, 5] = complex(float("nan"), 0.0)
    got = []
    with pytest.raises(InvariantError, match=r"a_blocks\[1\]"):
        for out in iter_hs_kpoints(ps, _pol("int8"), depth=3):
            got.append(out)
    assert len(got) == 2
    # the lanes were released: a new batch runs normally
    ps[2].a_blocks[1][3, 5] = 0.0
    assert len(list(iter_hs_kpoints(ps, _pol("int8"), depth=3))) == 6


def test_concurrent_calls_on_one_context_keep_their_engines():
    # two threads share process-wide context slot 0 with different engines:
    # every call must run on its own engine (settings + call are atomic per
    # context: _lib.using / CtxCall), so each result equals, bit for bit, the
    # serial result of its engine (_lib.py context races)
    import threading

    p = generate(ProblemSpec(Dims(3, 16, 120), seed=31, nonhpd_fraction=0.3))
    pols = {"int8": GpuPolicy(engine="int8"), "dmma": GpuPolicy(engine="dmma")}
    want = {k: build_hs(p, pol) for k, pol in pols.items()}
    assert not np.array_equal(want["int8"].h.matrix, want["dmma"].h.matrix)  # the engines are distinguishable
    errors = []

    def worker(k):
        try:
            for _ in range(12):
                out = build_hs(p, pols[k])
                if not (np.array_equal(out.h.matrix, want[k].h.matrix)
                        and np.array_equal(out.s.matrix, want[k].s.matrix)):
                    errors.append(k)
        except Exception as exc:  # noqa: BLE001
            errors.append(repr(exc))

    threads = [threading.Thread(target=worker, args=(k,)) for k in ("int8", "dmma", "int8", "dmma")]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("engine", ["auto", "dmma"])
def test_lower_only_outputs_leave_the_upper_triangle_untouched(engine):
    # HSB_OPT_LOWER_ONLY (the triangle-packed exchange's partials): the lower
    # triangle equals the FULL build's, the diagonal is real, and not one byte
    # of the strict upper triangle is written
    import torch

    from paper_1611_00606_b200 import DeviceProblem, build_hs_device

    p = generate(ProblemSpec(Dims(4, 20, 300), seed=32, nonhpd_fraction=0.25))
    dp = DeviceProblem.from_instance(p)
    pol = GpuPolicy(engine=engine)
    hf, sf, _, _, _ = build_hs_device(dp, policy=pol)
    n = p.dims.n_g
    sentinel = complex(123.0, -7.0)
    h = torch.full((n, n), sentinel, dtype=torch.complex128, device=dp.a_stack.device)
    s = torch.full_like(h, sentinel)
    build_hs_device(dp, h, s, pol, lower_only=True)
    torch.cuda.synchronize()
    for got, full in ((h, hf), (s, sf)):
        g = got.cpu().numpy().T  # column-major matrix
        f = full.cpu().numpy().T
        low = np.tril_indices(n)
        up = np.triu_indices(n, 1)
        assert np.array_equal(g[low], f[low])
        assert np.all(g[up] == sentinel)
        assert np.all(np.diagonal(g).imag == 0)


@pytest.mark.parametrize("cm", ["3m", "int8"])
def test_zero_columns_atoms_and_tiny_entries(cm):
    # degenerate data the per-column scaling of the INT8 engine must survive:
    # all-zero G columns of A and B (column maximum 0), an atom whose blocks
    # are all zero, and a column whose entries are 1e-200 (exponent far below
    # the others); both engines against the oracle
    p = generate(ProblemSpec(Dims(4, 25, 700), seed=77, nonhpd_fraction=0.25))
    for blocks in (p.a_blocks, p.b_blocks):
        for blk in blocks:
            blk[:, [0, 5, 699]] = 0.0
            blk[:, 17] *= 1e-200
    p.a_blocks[2][:] = 0.0
    p.b_blocks[2][:] = 0.0
    out = build_hs(p, _pol(cm))
    ref = alg1.build_hs_cpu(p)
    assert rel_frob_error(out.h.matrix, ref["h"]) < 1e-14
    assert rel_frob_error(out.s.matrix, ref["s"]) < 1e-14
    for c in (0, 5, 699):
        assert not np.any(out.h.matrix[:, c]) and not np.any(out.s.matrix[:, c])
    # the tiny column keeps its relative accuracy (per-column scaling)
    assert np.linalg.norm(out.s.matrix[:, 17] - ref["s"][:, 17]) <= 1e-13 * np.linalg.norm(ref["s"][:, 17])


@pytest.mark.parametrize("cm", ["3m", "int8"])
@pytest.mark.parametrize("dims", [Dims(1, 64, 256), Dims(2, 64, 512), Dims(2, 64, 257), Dims(3, 43, 255),
                                  Dims(2, 225, 300), Dims(1, 1, 1)])
def test_tile_boundaries(dims, cm):
    # N_G and K exactly on / one past the 256-wide INT8 tiles and 128-byte k
    # chunks, N_L above the 128-row V-product tiles, and the 1 x 1 x 1 corner
    p = generate(ProblemSpec(dims, seed=dims.n_g + dims.n_l, nonhpd_fraction=0.5))
    out = build_hs(p, _pol(cm))
    ref = alg1.build_hs_cpu(p)
    assert rel_frob_error(out.h.matrix, ref["h"]) < 1e-14
    assert rel_frob_error(out.s.matrix, ref["s"]) < 1e-14
    assert (out.split.hpd, out.split.nonhpd) == (ref["hpd"], ref["nonhpd"])


def test_wide_gemm_work_items_match_oracle():
    # the opt-in wide INT8 GEMM (HSB_OZ_WIDE: two row tiles per CTA pair, read
    # once per process, hence a subprocess): odd tile counts, slabs, both
    # contractions, against the oracle and bitwise against the default kernel
    import os
    import subprocess
    import sys

    from conftest import ROOT

    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "from oracle import alg1\n"
        "from paper_1611_00606_b200 import Dims, GpuPolicy, ProblemSpec, build_hs, generate, rel_frob_error\n"
        "for dims in (Dims(3, 49, 1301), Dims(9, 121, 700), Dims(70, 121, 300)):\n"
        "    p = generate(ProblemSpec(dims, seed=5, nonhpd_fraction=0.3))\n"
        "    o = build_hs(p, GpuPolicy(engine='int8'))\n"
        "    r = alg1.build_hs_cpu(p)\n"
        "    np.save('/tmp/wide_%%d_h.npy' %% dims.n_g, o.h.matrix)\n"
        "    print(rel_frob_error(o.h.matrix, r['h']), rel_frob_error(o.s.matrix, r['s']))\n" % str(ROOT))
    env = dict(os.environ, HSB_OZ_WIDE="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    errs = [float(x) for line in out.stdout.split("\n") if line.strip() for x in line.split()]
    assert len(errs) == 6 and max(errs) < 1e-14, errs
    # the default kernel gives the same bits (same residues, same reconstruction)
    for dims in (Dims(3, 49, 1301), Dims(9, 121, 700), Dims(70, 121, 300)):
        p = generate(ProblemSpec(dims, seed=5, nonhpd_fraction=0.3))
        assert np.array_equal(build_hs(p, GpuPolicy(engine="int8")).h.matrix, np.load("/tmp/wide_%d_h.npy" % dims.n_g))
