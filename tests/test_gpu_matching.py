"""Matching-coefficient kernel (csrc/match_kernel.cu) against the scipy-based
CPU restatement (oracle/matching.py), and the physical entry point
(atoms/types, lmax, G set, radial data, T -> H, S) against the oracle's
Algorithm 1 fed with the oracle's coefficients.  Tolerance 1e-12 on the
coefficients, 1e-10 on H and S (north star)."""

import numpy as np
import pytest
import torch

from oracle import alg1
from oracle import matching as om
from paper_1611_00606_b200 import Dims, ProblemInstance, rel_frob_error
from paper_1611_00606_b200.physics import (
    build_hs_physical, match_coeffs_device, synthetic_system, synthetic_t_matrices,
)

pytestmark = pytest.mark.gpu


def _oracle(system, k, g):
    return om.matching_coeffs(system.lattice.vectors, system.positions, system.types,
                              [s.rmt for s in system.species], system.radial_table(), system.lmax, k, g)


@pytest.mark.parametrize("n_atoms,n_types,lmax,ng,kpt", [
    (2, 1, 6, 500, (0.0, 0.0, 0.0)),     # C1 shape, Gamma point (K = 0 column present)
    (8, 2, 8, 3000, (0.25, -0.125, 0.5)),
    (3, 3, 10, 700, (0.1, 0.2, 0.3)),
    (1, 1, 0, 50, (0.0, 0.0, 0.0)),
    (4, 2, 14, 300, (0.5, 0.5, 0.5)),
])
def test_match_kernel_against_oracle(n_atoms, n_types, lmax, ng, kpt):
    system, _, kmax, _ = synthetic_system(n_atoms, n_types, lmax, ng, seed=lmax + n_atoms)
    from paper_1611_00606_b200.physics import gvector_set
    g = gvector_set(system.lattice, kpt, kmax)
    a_d, b_d = match_coeffs_device(system, kpt, g)
    torch.cuda.synchronize()
    a = a_d.cpu().numpy().T
    b = b_d.cpu().numpy().T
    ra, rb = _oracle(system, kpt, g)
    assert rel_frob_error(a, ra) < 1e-12
    assert rel_frob_error(b, rb) < 1e-12
    # elementwise too (relative to the column scale)
    assert np.max(np.abs(a - ra)) < 1e-12 * (1 + np.max(np.abs(ra)))


@pytest.mark.parametrize("engine", ["int8", "dmma"])
@pytest.mark.parametrize("lmax,kpt", [(8, (0.0, 0.0, 0.0)), (10, (0.1, 0.2, 0.3))])
def test_physical_build_matches_oracle_pipeline(engine, lmax, kpt):
    # physical coefficients span many orders of magnitude within a G column
    # (j_l(KR) ~ (KR)^l / (2l+1)!!): the INT8 engine's per-column scaling
    # must still meet the north star's 1e-10
    from paper_1611_00606_b200 import GpuPolicy

    system, k, kmax, g = synthetic_system(4, 2, lmax, 900, seed=3, kpt_frac=kpt)
    t_aa, t_ab, t_bb = synthetic_t_matrices(system, seed=3, nonhpd_fraction=0.25)
    h, s, split, t, info = build_hs_physical(system, k, g, t_aa, t_ab, t_bb, policy=GpuPolicy(engine=engine))
    torch.cuda.synchronize()
    ra, rb = _oracle(system, k, g)
    n_l, n_g = system.n_l, len(g)
    p = ProblemInstance(Dims(system.n_atoms, n_l, n_g))
    for al in range(system.n_atoms):
        p.a_blocks.append(np.asfortranarray(ra[al * n_l:(al + 1) * n_l]))
        p.b_blocks.append(np.asfortranarray(rb[al * n_l:(al + 1) * n_l]))
    p.t_aa, p.t_ab, p.t_bb, p.u_norms = t_aa, t_ab, t_bb, system.u_norms()
    ref = alg1.build_hs_cpu(p)
    assert (split.hpd, split.nonhpd) == (ref["hpd"], ref["nonhpd"])
    assert rel_frob_error(h.cpu().numpy().T, ref["h"]) < 1e-10
    assert rel_frob_error(s.cpu().numpy().T, ref["s"]) < 1e-10


@pytest.mark.parametrize("engine", ["int8", "dmma"])
def test_physical_build_host_outputs_match_device(engine):
    # the north-star entry point with H and S streamed to host memory (lower
    # triangles + host mirror on the INT8 path) equals the device-resident build
    from paper_1611_00606_b200 import GpuPolicy

    system, k, kmax, g = synthetic_system(5, 2, 8, 1300, seed=5)
    t_aa, t_ab, t_bb = synthetic_t_matrices(system, seed=5, nonhpd_fraction=0.2)
    pol = GpuPolicy(engine=engine)
    h, s, split, _, _ = build_hs_physical(system, k, g, t_aa, t_ab, t_bb, policy=pol)
    hh, sh, split_h, t, _ = build_hs_physical(system, k, g, t_aa, t_ab, t_bb, policy=pol, host_outputs=True)
    torch.cuda.synchronize()
    assert isinstance(hh, np.ndarray) and hh.shape == (len(g), len(g))
    assert (split.hpd, split.nonhpd) == (split_h.hpd, split_h.nonhpd)
    for name, a, b in (("H", hh, h.cpu().numpy().T), ("S", sh, s.cpu().numpy().T)):
        bad = np.argwhere(a != b)
        assert len(bad) == 0, (f"{name}: {len(bad)} entries differ ({int(np.sum(bad[:, 0] < bad[:, 1]))} above the "
                               f"diagonal), rows {bad[:, 0].min()}..{bad[:, 0].max()}, cols {bad[:, 1].min()}.."
                               f"{bad[:, 1].max()}, max |diff| {np.max(np.abs(a - b)):.3e}, first {bad[:4].tolist()}")
    assert t["d2h_bytes"] > 0


@pytest.mark.parametrize("engine,depth", [("int8", 3), ("dmma", 2), ("int8", 1)])
def test_physical_kpoint_pipeline_equals_serial(engine, depth):
    # config C5 from physical inputs: distinct k-points (so distinct, ragged G
    # sets) through the pipelined iterator equal serial build_hs_physical calls
    # bit for bit, in order; one k-point is also checked against the oracle
    from paper_1611_00606_b200 import GpuPolicy
    from paper_1611_00606_b200.physics import gvector_set, iter_hs_physical_kpoints

    system, _, kmax, _ = synthetic_system(4, 2, 6, 900, seed=11)
    t_aa, t_ab, t_bb = synthetic_t_matrices(system, seed=11, nonhpd_fraction=0.25)
    kpts = [np.array(k) for k in [(0.0, 0.0, 0.0), (0.5, 0.25, 0.0), (0.125, -0.375, 0.25), (0.5, 0.5, 0.5),
                                   (-0.25, 0.0, 0.125)]]
    gsets = [gvector_set(system.lattice, k, kmax) for k in kpts]
    assert len({g.shape[0] for g in gsets}) > 1  # ragged sizes
    pol = GpuPolicy(engine=engine)
    got = list(iter_hs_physical_kpoints(system, kpts, gsets, t_aa, t_ab, t_bb, policy=pol, depth=depth))
    assert len(got) == len(kpts)
    for (hh, sh, split, t, _), k, g in zip(got, kpts, gsets):
        h, s, split_s, _, _ = build_hs_physical(system, k, g, t_aa, t_ab, t_bb, policy=pol, host_outputs=True)
        assert hh.shape == (len(g), len(g))
        assert (split.hpd, split.nonhpd) == (split_s.hpd, split_s.nonhpd)
        assert np.array_equal(hh, h) and np.array_equal(sh, s)
    a, b = _oracle(system, kpts[2], gsets[2])
    n_l = system.n_l
    p = ProblemInstance(Dims(system.n_atoms, n_l, len(gsets[2])))
    p.a_blocks = [np.asfortranarray(a[i * n_l:(i + 1) * n_l]) for i in range(system.n_atoms)]
    p.b_blocks = [np.asfortranarray(b[i * n_l:(i + 1) * n_l]) for i in range(system.n_atoms)]
    p.t_aa, p.t_ab, p.t_bb, p.u_norms = t_aa, t_ab, t_bb, system.u_norms()
    ref = alg1.build_hs_cpu(p)
    assert (got[2][2].hpd, got[2][2].nonhpd) == (ref["hpd"], ref["nonhpd"])
    assert rel_frob_error(got[2][0], ref["h"]) < 1e-10
    assert rel_frob_error(got[2][1], ref["s"]) < 1e-10


def test_physical_kpoint_pipeline_rejects_mismatched_lists():
    from paper_1611_00606_b200 import InputError
    from paper_1611_00606_b200.physics import iter_hs_physical_kpoints

    system, k, _, g = synthetic_system(2, 1, 2, 100, seed=1)
    t = synthetic_t_matrices(system, seed=1)
    with pytest.raises(InputError):
        list(iter_hs_physical_kpoints(system, [k, k], [g], *t))


@pytest.mark.parametrize("lmax,ng,nonhpd", [(8, 1500, 0.25), (10, 3000, 0.0)])
def test_physical_build_fused_residues_match_the_standalone_passes(lmax, ng, nonhpd):
    # hsb_build_hs_physical: the matching kernel writes the INT8 engine's left
    # operands (column exponents, A and diag(u) B residue planes) as it
    # generates each G column; the build must equal, bit for bit, the
    # standalone path (coefficients to HBM, then the exponent and residue
    # passes over the stored stacks)
    from paper_1611_00606_b200 import DeviceProblem, GpuPolicy, build_hs_device
    from paper_1611_00606_b200.physics import _device_t

    system, k, kmax, g = synthetic_system(6, 3, lmax, ng, seed=lmax, kpt_frac=(0.2, -0.1, 0.3))
    t_aa, t_ab, t_bb = synthetic_t_matrices(system, seed=4, nonhpd_fraction=nonhpd)
    pol = GpuPolicy()
    h1, s1, sp1, t1, _ = build_hs_physical(system, k, g, t_aa, t_ab, t_bb, policy=pol)
    a, b = match_coeffs_device(system, k, g)
    dp = DeviceProblem(Dims(system.n_atoms, system.n_l, len(g)), a, b,
                       *_device_t(system, t_aa, t_ab, t_bb, a.device))
    h2, s2, sp2, t2, _ = build_hs_device(dp, policy=pol)
    torch.cuda.synchronize()
    assert (sp1.hpd, sp1.nonhpd) == (sp2.hpd, sp2.nonhpd)
    assert torch.equal(h1, h2) and torch.equal(s1, s2)
    assert t1["launches"] < t2["launches"]  # the exponent and A / UB residue passes are gone


def test_dmma_physical_builds_are_bitwise_repeatable():
    # regression: the DMMA kernels released a pipeline stage before their last
    # shared-memory loads had completed (the arrive does not wait for LDS in
    # flight), so the first builds of a new shape occasionally had a few wrong
    # rows in one warp's sub-tile (probes/stress_dmma_phys.py).  Device,
    # streamed-host and staged-host builds of one input must agree bit for bit.
    from paper_1611_00606_b200 import GpuPolicy

    system, k, kmax, g = synthetic_system(4, 2, 10, 2100, seed=3)
    t = synthetic_t_matrices(system, seed=3, nonhpd_fraction=0.2)
    pol, pol_staged = GpuPolicy(engine="dmma"), GpuPolicy(engine="dmma", pinned_outputs=False)
    ref = None
    for _ in range(3):
        for kind in ("device", "host", "staged"):
            if kind == "device":
                h, s, *_ = build_hs_physical(system, k, g, *t, policy=pol)
                torch.cuda.synchronize()
                h, s = h.cpu().numpy().T, s.cpu().numpy().T
            else:
                h, s, *_ = build_hs_physical(system, k, g, *t, policy=pol if kind == "host" else pol_staged,
                                             host_outputs=True)
            if ref is None:
                ref = (h.copy(), s.copy())
            assert np.array_equal(h, ref[0]) and np.array_equal(s, ref[1]), kind
