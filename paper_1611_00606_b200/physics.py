"""Physical front end: atoms/types, lmax, G-vector set, radial data -> H, S.

The reference takes the matching coefficients A, B as synthetic random inputs
(probgen.py:131-132); the north star asks for them to be
*generated* from the FLAPW basis (Rayleigh expansion of the
interstitial plane wave matched in value and slope at the muffin-tin radius).
This module holds the host side of that: the G-vector enumeration (done once,
on the host, shared by the GPU kernel and the CPU oracle so G and lm indexing
are bit-exact by construction), synthetic systems of the BASELINE shapes,
and ``build_hs_physical`` which runs ``hsb_match_coeffs`` (csrc/match_kernel.cu)
and then the H/S pipeline, all on the device.

Conventions, for atom alpha of type t at
Cartesian tau_alpha, K = k + G (Cartesian, 1/bohr):

    c_lm   = (4 pi / sqrt(Omega)) i^l exp(i K . tau_alpha) conj(Y_lm(K^))
    A_lm   = c_lm [ j_l(KR) udot'_l - K j_l'(KR) udot_l ] / D_l
    B_lm   = c_lm [ K j_l'(KR) u_l  - j_l(KR) u'_l      ] / D_l
    D_l    = u_l udot'_l - udot_l u'_l        (radial values at R_t)

Y_lm complex with the Condon-Shortley phase (scipy.special.sph_harm_y,
theta polar); lm row index L = l^2 + l + m; rows of the stacked A/B are
(atom, L) atom-major; columns follow the G list order.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .hs_types import Dims, InputError
from .instances import _hermitian_with_spectrum, _gauss


@dataclass(frozen=True)
class Lattice:
    """Real-space lattice vectors as rows (bohr)."""

    vectors: np.ndarray

    @property
    def volume(self) -> float:
        return float(abs(np.linalg.det(self.vectors)))

    @property
    def reciprocal(self) -> np.ndarray:
        """Rows b_i with a_i . b_j = 2 pi delta_ij (1/bohr)."""
        return 2.0 * math.pi * np.linalg.inv(self.vectors).T

    @classmethod
    def cubic(cls, a: float) -> "Lattice":
        return cls(np.eye(3) * float(a))

    @classmethod
    def orthorhombic(cls, a: float, b: float, c: float) -> "Lattice":
        return cls(np.diag([float(a), float(b), float(c)]))


@dataclass
class Species:
    """Muffin-tin radius and radial boundary data for l = 0..lmax.

    ``radial[l] = (u_l(R), u_l'(R), udot_l(R), udot_l'(R))``; ``udot_norm[l]``
    is ||udot_l|| (the U of Alg. 1 line 14, unsquared, builder.py:124-131).
    """

    rmt: float
    radial: np.ndarray      # (lmax+1, 4)
    udot_norm: np.ndarray   # (lmax+1,)


@dataclass
class PhysicalSystem:
    lattice: Lattice
    positions: np.ndarray   # (n_atoms, 3) Cartesian, bohr
    types: np.ndarray       # (n_atoms,) int
    species: list
    lmax: int

    @property
    def n_atoms(self) -> int:
        return int(self.positions.shape[0])

    @property
    def n_l(self) -> int:
        return (self.lmax + 1) ** 2

    def radial_table(self) -> np.ndarray:
        """(n_types, lmax+1, 4) float64."""
        return np.ascontiguousarray(np.stack([np.asarray(s.radial, dtype=np.float64) for s in self.species]))

    def u_norms(self) -> list:
        """Per-atom U rows: ||udot_l|| repeated over m (lm order L = l^2 + l + m)."""
        lidx = l_of_lm(self.lmax)
        return [np.asarray(self.species[t].udot_norm, dtype=np.float64)[lidx] for t in self.types]


def l_of_lm(lmax: int) -> np.ndarray:
    """l for each row L = l^2 + l + m, m = -l..l."""
    return np.concatenate([np.full(2 * l + 1, l, dtype=np.int64) for l in range(lmax + 1)])


def gvector_set(lattice: Lattice, kpt_frac, kmax: float) -> np.ndarray:
    """Integer triples n with |k + n.B| <= kmax, lexicographic (n1, n2, n3) order.

    Computed once on the host; the GPU kernel and the CPU oracle both index
    columns by this exact list (bit-exact G ordering by construction).
    """
    b = lattice.reciprocal
    k = np.asarray(kpt_frac, dtype=np.float64)
    # bound |n_i| via the distance between lattice planes of the reciprocal lattice
    a = lattice.vectors
    nmax = [int(math.ceil(kmax * np.linalg.norm(a[i]) / (2 * math.pi) + abs(k[i]))) + 1 for i in range(3)]
    rng = [np.arange(-n, n + 1) for n in nmax]
    n1, n2, n3 = np.meshgrid(*rng, indexing="ij")
    trip = np.stack([n1.ravel(), n2.ravel(), n3.ravel()], axis=1)
    kc = (trip + k) @ b
    keep = np.einsum("ij,ij->i", kc, kc) <= kmax * kmax
    out = trip[keep]
    order = np.lexsort((out[:, 2], out[:, 1], out[:, 0]))
    return np.ascontiguousarray(out[order].astype(np.int32))


def synthetic_system(n_atoms: int, n_types: int, lmax: int, target_ng: int, seed: int = 0,
                     kmax: float = 4.0, kpt_frac=(0.0, 0.0, 0.0)):
    """Near-cubic cell sized so |k+G| <= kmax holds target_ng (+-1 %) vectors.

    The axes are in slightly incommensurate ratios (1 : 1.0137 : 0.9871) so the
    G-count grows smoothly with the cell size instead of in cubic shells.

    Atoms at seeded uniform fractional positions, types round-robin,
    R_t in [2.0, 2.4] bohr, seeded radial values with |D| bounded away from 0.
    Returns (system, kpt_frac, kmax, gset).
    """
    rng = np.random.Generator(np.random.Philox(seed))
    # N_G ~ (4 pi / 3) kmax^3 Omega / (2 pi)^3 -> a from the target, then bisect on the exact count
    ratios = (1.0, 1.0137, 0.9871)

    def cell(a):
        return Lattice.orthorhombic(*(a * r for r in ratios))

    a0 = 2 * math.pi / kmax * (3 * target_ng / (4 * math.pi)) ** (1 / 3)
    lo, hi = 0.8 * a0, 1.2 * a0
    best = None
    for _ in range(60):
        a = 0.5 * (lo + hi)
        n = gvector_set(cell(a), kpt_frac, kmax).shape[0]
        if best is None or abs(n - target_ng) < abs(best[1] - target_ng):
            best = (a, n)
        if n == target_ng:
            break
        if n < target_ng:
            lo = a
        else:
            hi = a
    a = best[0]
    lattice = cell(a)
    frac = rng.uniform(0.0, 1.0, size=(n_atoms, 3))
    positions = frac @ lattice.vectors
    types = np.arange(n_atoms) % n_types
    species = []
    for t in range(n_types):
        rmt = 2.0 + 0.4 * t / max(1, n_types - 1)
        rad = np.empty((lmax + 1, 4))
        for l in range(lmax + 1):
            while True:
                u, du, ud, dud = rng.uniform(0.2, 1.5), rng.uniform(-1.0, 1.0), rng.uniform(-0.8, 0.8), rng.uniform(0.5, 2.0)
                if abs(u * dud - ud * du) > 0.1:
                    break
            rad[l] = (u, du, ud, dud)
        species.append(Species(rmt, rad, rng.uniform(0.5, 1.5, size=lmax + 1)))
    system = PhysicalSystem(lattice, positions, types.astype(np.int64), species, lmax)
    gset = gvector_set(lattice, kpt_frac, kmax)
    return system, np.asarray(kpt_frac, dtype=np.float64), kmax, gset


def synthetic_t_matrices(system: PhysicalSystem, seed: int = 0, nonhpd_fraction: float = 0.0):
    """Per-atom T_AA, T_AB, T_BB (probgen conventions, probgen.py:95-137)."""
    rng = np.random.Generator(np.random.Philox(seed + 7919))
    n_a, n_l = system.n_atoms, system.n_l
    flagged = set(rng.permutation(n_a)[: round(nonhpd_fraction * n_a)].tolist())
    scale = 1.0 / math.sqrt(n_l)
    t_aa, t_ab, t_bb = [], [], []
    for a in range(n_a):
        t_ab.append(_gauss(rng, n_l, n_l, scale))
        t_aa.append(_hermitian_with_spectrum(rng, n_l, 0.5, 2.0, a in flagged))
        t_bb.append(_hermitian_with_spectrum(rng, n_l, 0.5, 2.0, False))
    return t_aa, t_ab, t_bb


# ------------------------------------------------------------------ device side

def _phys_struct(system: PhysicalSystem, kpt, gset):
    g = np.ascontiguousarray(gset, dtype=np.int32)
    if g.ndim != 2 or g.shape[1] != 3 or g.shape[0] < 1:
        raise InputError("gset must be an (n_g, 3) integer array with n_g >= 1")
    tau = np.ascontiguousarray(system.positions, dtype=np.float64)
    types = np.ascontiguousarray(system.types, dtype=np.int32)
    n_types = len(system.species)
    if types.min() < 0 or types.max() >= n_types:
        raise InputError("atom type index out of range")
    rmt = np.ascontiguousarray([s.rmt for s in system.species], dtype=np.float64)
    radial = system.radial_table()
    if radial.shape != (n_types, system.lmax + 1, 4):
        raise InputError("radial table must be (n_types, lmax+1, 4)")
    d = radial[..., 0] * radial[..., 3] - radial[..., 2] * radial[..., 1]
    if np.any(d == 0) or not np.all(np.isfinite(radial)):
        raise InputError("radial data must be finite with a non-zero Wronskian D_l")
    s = _lib.HsbPhys()
    s.n_atoms, s.n_g, s.lmax, s.n_types = system.n_atoms, g.shape[0], system.lmax, n_types
    s.gvec = g.ctypes.data
    s.tau = tau.ctypes.data
    s.type_of = types.ctypes.data
    s.rmt = rmt.ctypes.data
    s.radial = radial.ctypes.data
    for i in range(3):
        s.kpt[i] = float(kpt[i])
    rec = system.lattice.reciprocal
    for i in range(9):
        s.recip[i] = float(rec.flat[i])
    s.omega = system.lattice.volume
    return s, (g, tau, types, rmt, radial)


def match_coeffs_device(system: PhysicalSystem, kpt, gset, device: int = 0, stream=None, slot: int = 0,
                        out=None):
    """A, B stacks on the device: torch complex128 (n_g, n_atoms*n_l) tensors
    (= column-major K x n_g), generated by the sm_100a matching kernel.
    ``out`` = (a, b) writes into caller-owned tensors of that shape; ``slot``
    picks the library context whose workspace stages the small inputs."""
    import torch

    lib = _lib.load()
    ctx = _lib.context(device, slot=slot)
    dev = torch.device("cuda", device)
    n_g, k = int(gset.shape[0]), system.n_atoms * system.n_l
    if out is None:
        a = torch.empty((n_g, k), dtype=torch.complex128, device=dev)
        b = torch.empty_like(a)
    else:
        a, b = out
        for t in (a, b):
            if tuple(t.shape) != (n_g, k) or t.dtype != torch.complex128 or not t.is_contiguous() or t.device != dev:
                raise InputError(f"out tensors must be contiguous complex128 of shape ({n_g}, {k}) on {dev}")
    s, _keep = _phys_struct(system, kpt, gset)
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    _lib.check(lib.hsb_match_coeffs(ctx, ctypes.c_void_p(stream.cuda_stream), ctypes.byref(s), a.data_ptr(),
                                    b.data_ptr(), k), ctx)
    return a, b


def _device_t(system: PhysicalSystem, t_aa, t_ab, t_bb, dev):
    """T_AA, T_AB, T_BB as (n_atoms, n_l, n_l) device stacks and U (K,)."""
    import torch

    n_a, n_l = system.n_atoms, system.n_l

    def mats(blocks):
        if len(blocks) != n_a:
            raise InputError(f"expected {n_a} T blocks, got {len(blocks)}")
        host = np.stack([np.asarray(x, dtype=np.complex128).T for x in blocks])
        if host.shape != (n_a, n_l, n_l):
            raise InputError(f"T blocks must be {n_l} x {n_l}")
        return torch.from_numpy(np.ascontiguousarray(host)).to(dev)

    u = torch.from_numpy(np.concatenate(system.u_norms())).to(dev)
    return mats(t_aa), mats(t_ab), mats(t_bb), u


def build_hs_physical(system: PhysicalSystem, kpt, gset, t_aa, t_ab, t_bb, policy=None,
                      force_nonhpd: bool = False, host_outputs: bool = False):
    """North-star entry point: physical inputs in, H and S out (device tensors,
    or column-major numpy arrays with ``host_outputs``).

    Matching coefficients are generated on the device and consumed in place
    by the H/S pipeline (no host round trip), in one library call
    (hsb_build_hs_physical): with the INT8 engine the matching kernel also
    writes the exponents and residue planes of A and diag(u) B that S and H
    start from.  Returns (H, S, SplitCounts, timings,
    atom_info) like ``build_hs_device``.
    """
    import torch

    from .pipeline import DeviceProblem, GpuPolicy, build_hs_device

    pol = policy if isinstance(policy, GpuPolicy) else GpuPolicy()
    dev = torch.device("cuda", pol.device)
    dims = Dims(system.n_atoms, system.n_l, int(gset.shape[0]))
    a = torch.empty((dims.n_g, dims.k), dtype=torch.complex128, device=dev)
    b = torch.empty_like(a)
    dp = DeviceProblem(dims, a, b, *_device_t(system, t_aa, t_ab, t_bb, dev))
    phys, _keep = _phys_struct(system, kpt, gset)
    return build_hs_device(dp, policy=pol, force_nonhpd=force_nonhpd, host_outputs=host_outputs, phys=phys)


def iter_hs_physical_kpoints(system: PhysicalSystem, kpts, gsets, t_aa, t_ab, t_bb, policy=None,
                             force_nonhpd: bool = False, depth: int = 3):
    """Yield (H, S, SplitCounts, timings, atom_info) of ``build_hs_physical(...,
    host_outputs=True)`` for each k-point in order (BASELINE config C5 from
    physical inputs), pipelined on one GPU.

    The T matrices and U are k-independent: they are uploaded once and shared
    by every k-point.  ``depth`` lanes (host threads, each with its own
    library context, CUDA stream and A/B buffers sized for the largest G set)
    run in turn: lane i % depth generates k-point i's A and B in its buffers
    and builds H and S from them; the contractions run in k-point order on the
    SMs (compute events, as in ``pipeline.iter_hs_kpoints``) while earlier
    k-points' H and S stream to pinned host memory.  Every result equals the
    serial ``build_hs_physical`` of that k-point bit for bit.
    """
    import torch

    from .pipeline import DeviceProblem, GpuPolicy, _lane_pipeline, build_hs_device

    pol = policy if isinstance(policy, GpuPolicy) else GpuPolicy()
    if int(depth) != depth or depth < 1:
        raise InputError(f"depth must be a positive integer, got {depth!r}")
    kpts, gsets = list(kpts), list(gsets)
    if len(kpts) != len(gsets):
        raise InputError(f"{len(kpts)} k-points but {len(gsets)} G sets")
    if not kpts:
        return
    dev = torch.device("cuda", pol.device)
    tdev = _device_t(system, t_aa, t_ab, t_bb, dev)
    k = system.n_atoms * system.n_l
    n_max = max(int(g.shape[0]) for g in gsets)
    depth = min(int(depth), len(kpts))
    bufs = [(torch.empty((n_max, k), dtype=torch.complex128, device=dev),
             torch.empty((n_max, k), dtype=torch.complex128, device=dev)) for _ in range(depth)]
    torch.cuda.synchronize(dev)  # T uploads and buffers ready before the lanes' streams use them

    def run(i, slot, stream, order):
        n_g = int(gsets[i].shape[0])
        a, b = bufs[slot][0][:n_g], bufs[slot][1][:n_g]
        dp = DeviceProblem(Dims(system.n_atoms, system.n_l, n_g), a, b, *tdev)
        phys, _keep = _phys_struct(system, kpts[i], gsets[i])
        return build_hs_device(dp, policy=pol, force_nonhpd=force_nonhpd, stream=stream, host_outputs=True,
                               slot=slot, order=order, phys=phys)

    if depth == 1:
        st = torch.cuda.current_stream(dev)
        for i in range(len(kpts)):
            yield run(i, 0, st, None)
        return
    yield from _lane_pipeline(len(kpts), depth, pol, n_max, run)
