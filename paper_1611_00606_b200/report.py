"""Per-section report of a GPU build: the paper's Table 5 on B200.

Mirrors ``hsgen.report`` (/root/reference/pkg/src/hsgen/report.py):

* ``summarize(ledger, peak_gflops)`` -> SectionReport per section in SECTIONS
  order (report.py:57-76);
* ``format_table`` -> the aligned text table (report.py:159-166);
* ``TABLE5`` -> the recorded NaCl K_max 4.0 breakdown on 2 x K20x + 16 cores
  (report.py:45-54).

The ledger fed here comes from ``build_hs`` and its seconds come from CUDA
events (pipeline.py).  ``B200_FP64_PEAK_GFLOPS`` is the measured DMMA peak
(profiles/fp64_peak_r01.jsonl), which replaces the reference's 2.6 TF
two-K20x peak as the efficiency denominator.
"""

from __future__ import annotations

from dataclasses import dataclass

from .hs_types import InputError
from .ledger import HEAVY_SECTIONS, SECTIONS, FlopLedger, section_flops
from .instances import preset_dims

#: Measured sustained FP64 DMMA peak of one B200 (GFLOP/s), probes/fp64_peak.cu.
B200_FP64_PEAK_GFLOPS = 36920.0
#: Peak the reference's recorded efficiencies were computed against (report.py:19-24).
PEAK_GFLOPS_2GPU = 2600.0
PEAK_GFLOPS_CPU = 256.0
PEAK_GFLOPS_COMBINED = PEAK_GFLOPS_2GPU + PEAK_GFLOPS_CPU


@dataclass(frozen=True)
class SectionReport:
    section: str
    seconds: float
    flops: int
    gflops_per_s: float | None
    efficiency: float | None


@dataclass(frozen=True)
class Table5Row:
    section: str
    seconds: float
    gflops_per_s: float


TABLE5 = (
    Table5Row("Loop 1", 2.27, 80.35), Table5Row("Loop 2", 2.62, 34.81), Table5Row("U norm", 0.23, 1.01),
    Table5Row("S1", 4.37, 1974.63), Table5Row("S2", 4.41, 1956.72), Table5Row("H1", 9.49, 1818.57),
    Table5Row("H2", 2.32, 1859.72), Table5Row("H3", 4.75, 1816.66),
)


def summarize(ledger: FlopLedger, peak_gflops: float = B200_FP64_PEAK_GFLOPS) -> list:
    """One SectionReport per section present, in Table-5 order; zero time -> None rates."""
    if not len(ledger):
        raise InputError("cannot summarize an empty ledger")
    if not peak_gflops > 0:
        raise InputError(f"peak_gflops must be positive, got {peak_gflops!r}")
    totals = ledger.section_totals()
    out = []
    for section in SECTIONS:
        if section not in totals:
            continue
        flops, seconds = totals[section]
        rate = flops / seconds / 1e9 if seconds > 0 else None
        out.append(SectionReport(section, seconds, flops, rate, None if rate is None else rate / peak_gflops))
    return out


def format_table(reports) -> str:
    lines = [f"{'Section':<10} {'Time':>12} {'Performance':>18} {'Efficiency':>12}"]
    for r in reports:
        perf = "-" if r.gflops_per_s is None else f"{r.gflops_per_s:.2f} GFlops/s"
        eff = "-" if r.efficiency is None else f"{r.efficiency:.2f}"
        lines.append(f"{r.section:<10} {r.seconds:>7.4f} secs {perf:>18} {eff:>12}")
    return "\n".join(lines)


def compare_with_table5(reports) -> str:
    """Side-by-side of a B200 breakdown and the paper's NaCl 4.0 Table 5."""
    paper = {r.section: r for r in TABLE5}
    lines = [f"{'Section':<8} {'paper s':>9} {'paper GF/s':>11} {'B200 s':>10} {'B200 GF/s':>11} {'B200 eff':>9}"]
    for r in reports:
        p = paper.get(r.section)
        lines.append(f"{r.section:<8} {p.seconds if p else float('nan'):>9.2f} "
                     f"{p.gflops_per_s if p else float('nan'):>11.2f} {r.seconds:>10.4f} "
                     f"{(r.gflops_per_s or 0):>11.1f} {(r.efficiency or 0):>9.3f}")
    return "\n".join(lines)


def heavy_fraction_of(ledger: FlopLedger) -> float:
    totals = ledger.section_totals()
    return sum(totals[s][0] for s in HEAVY_SECTIONS if s in totals) / max(1, ledger.total_flops())


def nacl_table5_dims():
    """Dimensions of the paper's Table-5 case (NaCl, K_max 4.0): 512 atoms, N_L 49, N_G 9273."""
    return preset_dims("NaCl", 4.0)


def model_seconds_at_peak(dims, nonhpd_count: int = 0, peak_gflops: float = B200_FP64_PEAK_GFLOPS) -> float:
    """Lower bound on one build's time at the given peak (model flops / peak)."""
    return sum(section_flops(dims, nonhpd_count).values()) / (peak_gflops * 1e9)
