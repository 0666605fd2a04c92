"""paper_1611_00606_b200 — B200-native H/S generation (arXiv 1611.00606, HSDLA).

Drop-in for the hot path of the reference package ``hsgen``: generating the
FLAPW Hamiltonian H and overlap S for one k-point.  The public names mirror
``hsgen`` (/root/reference/pkg/src/hsgen/__init__.py); every dense
contraction runs in hand-written sm_100a kernels in ``libhsb200.so``.

    from paper_1611_00606_b200 import generate, ProblemSpec, Dims, build_hs
    out = build_hs(generate(ProblemSpec(Dims(32, 121, 8000))))
"""

from .hs_types import (
    DimensionError,
    Dims,
    Fill,
    HermitianResult,
    InputError,
    InvariantError,
    SplitCounts,
    frobenius,
    hermitian_defect,
    hermitian_mirror_host,
    is_hermitian,
    rel_frob_error,
)
from .instances import (
    CONFIGS,
    PRESETS,
    Preset,
    ProblemInstance,
    ProblemSpec,
    generate,
    preset_dims,
    validate_instance,
)
from .ledger import (
    HEAVY_SECTIONS,
    SECTIONS,
    FlopLedger,
    FlopRecord,
    KernelKind,
    flops_of,
    heavy_fraction,
    section_flops,
    total_model_flops,
)
from .pipeline import (BuildOutput, DeviceProblem, GpuPolicy, build_hs, build_hs_device, build_hs_kpoints,
                       iter_hs_kpoints, pin_instance)
from .offload import ExecResult, run_partitioned
from .engine import int8_gemm_ops, int8_moduli

__version__ = "0.1.0"
