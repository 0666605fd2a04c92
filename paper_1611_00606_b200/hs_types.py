"""Value types of the drop-in boundary (host side, no GPU code).

Mirrors the public surface of the reference's ``hsgen.matcore``
(/root/reference/pkg/src/hsgen/matcore.py) so callers of ``build_hs`` see the
same names, fields and exception classes:

* ``Dims`` (matcore.py:28-44), the error hierarchy (matcore.py:16-25) --
  the reference's own classes whenever ``hsgen`` is importable,
* ``Fill`` / ``HermitianResult`` with ``check`` and ``mirrored``
  (matcore.py:47-49, 128-161),
* ``rel_frob_error`` — the parity metric ||a-b||_F / (1+||b||_F)
  (matcore.py:121-125) used by every parity test in ``tests/``.

Matrices are numpy complex128 column-major, as in the reference.
"""

from __future__ import annotations

import enum
import importlib
import importlib.util
import os
from dataclasses import dataclass

import numpy as np


def reference_module(name: str):
    """``hsgen.<name>`` of the reference package when it is importable (a
    caller switching to the drop-in has it installed), else None.  The
    drop-in then raises the reference's own exception classes and returns
    its ``BuildOutput``, so callers' ``except InvariantError`` (cli.py:161,
    199) and type checks keep working.  ``HSB200_STANDALONE=1`` disables it."""
    if os.environ.get("HSB200_STANDALONE"):
        return None
    try:
        if importlib.util.find_spec("hsgen") is None:
            return None
        return importlib.import_module(f"hsgen.{name}")
    except Exception:  # noqa: BLE001 -- a broken install is treated as absent
        return None


_REF_MATCORE = reference_module("matcore")

if _REF_MATCORE is not None:
    # the very classes of the reference (matcore.py:16-25)
    DimensionError = _REF_MATCORE.DimensionError
    InputError = _REF_MATCORE.InputError
    InvariantError = _REF_MATCORE.InvariantError
else:
    class DimensionError(ValueError):
        """Shapes of operands do not conform (matcore.DimensionError)."""

    class InputError(ValueError):
        """An operand value is invalid (matcore.InputError)."""

    class InvariantError(ValueError):
        """A declared invariant is violated (matcore.InvariantError)."""


@dataclass(frozen=True)
class Dims:
    """(n_atoms, n_l, n_g): atoms, (l, m) rows per atom block, basis size."""

    n_atoms: int
    n_l: int
    n_g: int

    def __post_init__(self):
        for name in ("n_atoms", "n_l", "n_g"):
            value = getattr(self, name)
            try:
                ok = int(value) == value and int(value) >= 1
            except (TypeError, ValueError):
                ok = False
            if not ok:
                raise InputError(f"{name} must be a positive integer, got {value!r}")
            object.__setattr__(self, name, int(value))

    @property
    def k(self) -> int:
        """Height of the stacked coefficient matrices, n_atoms * n_l."""
        return self.n_atoms * self.n_l


class Fill(enum.Enum):
    LOWER = "lower"
    FULL = "full"


def frobenius(m) -> float:
    return float(np.linalg.norm(np.asarray(m)))


def rel_frob_error(a, b) -> float:
    """||a - b||_F / (1 + ||b||_F) — the reference's parity metric."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise DimensionError(f"shape mismatch: {a.shape} vs {b.shape}")
    return frobenius(a - b) / (1.0 + frobenius(b))


def hermitian_defect(m) -> float:
    """max(|M - M^H|, |Im diag M|); 0 for an empty matrix."""
    m = np.asarray(m)
    if m.size == 0:
        return 0.0
    return max(float(np.abs(m - m.conj().T).max()), float(np.abs(np.diagonal(m).imag).max()))


def is_hermitian(m, tol: float = 1e-12) -> bool:
    return hermitian_defect(m) <= tol * (1.0 + frobenius(m))


def hermitian_mirror_host(m) -> np.ndarray:
    """Host copy of matcore.hermitian_mirror: upper := conj(lower), real diagonal.

    Only used on host-resident results (``HermitianResult.mirrored``); the
    device pipeline fuses the mirror into its epilogue.
    """
    m = np.asarray(m)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise DimensionError(f"hermitian_mirror needs a square matrix, got {m.shape}")
    low = np.tril(m, -1)
    out = low + low.conj().T + np.diag(np.diagonal(m).real)
    return np.asfortranarray(out.astype(np.complex128, copy=False))


@dataclass
class HermitianResult:
    """A square complex matrix and the triangle it is guaranteed to hold."""

    matrix: np.ndarray
    fill: Fill

    @property
    def order(self) -> int:
        return self.matrix.shape[0]

    def mirrored(self) -> "HermitianResult":
        if self.fill is Fill.FULL:
            return self
        return HermitianResult(hermitian_mirror_host(self.matrix), Fill.FULL)

    def check(self, tol: float = 1e-12) -> None:
        """Raise InvariantError unless the storage contract holds (matcore.py:148-161)."""
        m = self.matrix
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise InvariantError(f"result matrix must be square, got {m.shape}")
        if not np.isfinite(m).all():
            raise InvariantError("result matrix contains non-finite entries")
        bound = tol * (1.0 + frobenius(m))
        if m.size and float(np.abs(np.diagonal(m).imag).max()) > bound:
            raise InvariantError("diagonal imaginary parts exceed tolerance")
        if self.fill is Fill.FULL and m.size and float(np.abs(m - m.conj().T).max()) > bound:
            raise InvariantError("matrix is not Hermitian within tolerance")


@dataclass(frozen=True)
class SplitCounts:
    """Atoms routed to the Cholesky (hpd) and Hermitian-multiply (nonhpd) paths."""

    hpd: int
    nonhpd: int
