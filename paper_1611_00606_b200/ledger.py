"""Flop model and per-kernel ledger (host side).

Same vocabulary and integers as the reference so ledgers are comparable
record by record:

* ``KernelKind`` values and ``SECTIONS`` tags — kernels.py:26-38,
* ``flops_of`` — the paper's per-line annotations, kernels.py:51-85
  (complex MAC = 8 flops; HERK/HER2K/TRMM count the stored triangle only),
* ``FlopRecord`` / ``FlopLedger`` — kernels.py:88-139,
* ``section_flops`` / ``heavy_fraction`` — report.py:79-114.

``section_flops`` is also the *algorithmic* flop count that every
throughput and roofline number in this repository is quoted on.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

from .hs_types import Dims, InputError, InvariantError


class KernelKind(enum.Enum):
    GEMM = "gemm"
    HEMM = "hemm"
    HERK = "herk"
    HER2K = "her2k"
    TRMM = "trmm"
    POTRF = "potrf"
    DIAG_SCALE = "diag_scale"


SECTIONS = ("Loop 1", "Loop 2", "U norm", "S1", "S2", "H1", "H2", "H3")
HEAVY_SECTIONS = ("S1", "S2", "H1", "H2", "H3")

_ARITY = {
    KernelKind.GEMM: 3, KernelKind.HEMM: 2, KernelKind.HERK: 2, KernelKind.HER2K: 2,
    KernelKind.TRMM: 2, KernelKind.POTRF: 1, KernelKind.DIAG_SCALE: 2,
}


def _kind_of(kind) -> KernelKind:
    if isinstance(kind, KernelKind):
        return kind
    # accept the reference's own enum members (same .value strings)
    value = getattr(kind, "value", None)
    for k in KernelKind:
        if k.value == value:
            return k
    raise InputError(f"unknown kernel kind {kind!r}")


def flops_of(kind, dims) -> int:
    """Model flops of one kernel call; dims as in kernels.flops_of."""
    kind = _kind_of(kind)
    dims = tuple(int(d) for d in dims)
    if len(dims) != _ARITY[kind] or min(dims, default=0) < 0:
        raise InputError(f"bad dims {dims} for {kind.value}")
    if kind is KernelKind.GEMM:
        m, n, k = dims
        return 8 * m * n * k
    if kind is KernelKind.POTRF:
        return round(4 * dims[0] ** 3 / 3)
    a, b = dims
    per = {KernelKind.HEMM: 8 * a * a * b, KernelKind.HERK: 4 * b * a * a,
           KernelKind.HER2K: 8 * b * a * a, KernelKind.TRMM: 4 * a * a * b,
           KernelKind.DIAG_SCALE: 2 * a * b}
    return per[kind]


@dataclass(frozen=True)
class FlopRecord:
    kind: KernelKind
    dims: tuple
    flops: int
    seconds: float
    section: str

    def __post_init__(self):
        if self.section not in SECTIONS:
            raise InputError(f"unknown section tag {self.section!r}")
        if self.flops != flops_of(self.kind, self.dims):
            raise InvariantError(f"flops {self.flops} != flops_of({self.kind}, {self.dims})")
        if self.seconds < 0:
            raise InputError("seconds must be nonnegative")


class FlopLedger:
    """Ordered list of kernel invocations of one build."""

    def __init__(self):
        self.records: list[FlopRecord] = []

    def add(self, kind, dims, seconds: float, section: str) -> FlopRecord:
        kind = _kind_of(kind)
        dims = tuple(int(d) for d in dims)
        rec = FlopRecord(kind, dims, flops_of(kind, dims), float(seconds), section)
        self.records.append(rec)
        return rec

    def total_flops(self) -> int:
        return sum(r.flops for r in self.records)

    def total_seconds(self) -> float:
        return sum(r.seconds for r in self.records)

    def section_totals(self) -> dict:
        totals: dict[str, tuple[int, float]] = {}
        for r in self.records:
            f, s = totals.get(r.section, (0, 0.0))
            totals[r.section] = (f + r.flops, s + r.seconds)
        return totals

    def __len__(self) -> int:
        return len(self.records)

    def __iter__(self):
        return iter(self.records)


def section_flops(dims: Dims, nonhpd_count: int) -> dict:
    """Closed-form model flops per section (report.section_flops, report.py:79-105)."""
    n_a, n_l, n_g = dims.n_atoms, dims.n_l, dims.n_g
    if not 0 <= nonhpd_count <= n_a:
        raise InputError(f"nonhpd_count must be in [0, {n_a}], got {nonhpd_count}")
    k = n_a * n_l
    m = nonhpd_count
    h = n_a - m
    gemm_small = flops_of(KernelKind.GEMM, (n_l, n_g, n_l))
    hemm_small = flops_of(KernelKind.HEMM, (n_l, n_g))
    potrf_trmm = flops_of(KernelKind.POTRF, (n_l,)) + flops_of(KernelKind.TRMM, (n_l, n_g))
    return {
        "Loop 1": n_a * (gemm_small + hemm_small),
        "Loop 2": h * potrf_trmm + m * hemm_small,
        "U norm": flops_of(KernelKind.DIAG_SCALE, (k, n_g)),
        "S1": flops_of(KernelKind.HERK, (n_g, k)),
        "S2": flops_of(KernelKind.HERK, (n_g, k)),
        "H1": flops_of(KernelKind.HER2K, (n_g, k)),
        "H2": flops_of(KernelKind.GEMM, (n_g, n_g, m * n_l)) if m else 0,
        "H3": flops_of(KernelKind.HERK, (n_g, h * n_l)) if h else 0,
    }


def total_model_flops(dims: Dims, nonhpd_count: int = 0) -> int:
    return sum(section_flops(dims, nonhpd_count).values())


def heavy_fraction(dims: Dims, nonhpd_count: int) -> float:
    per = section_flops(dims, nonhpd_count)
    return sum(per[s] for s in HEAVY_SECTIONS) / sum(per.values())
