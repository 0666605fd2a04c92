"""Kernel-level drop-in: ``run_partitioned`` on the B200.

Reference: ``hsgen.executor.run_partitioned(kind, operands, policy)``
(/root/reference/pkg/src/hsgen/executor.py:185-225) with the operand tuples
of the serial kernels (executor.py:188-193):

* GEMM  ``(alpha, opa, a, opb, b, beta, c)``   — kernels.gemm (kernels.py:195-220)
* HERK  ``(alpha, a, beta, c)``               — kernels.herk (kernels.py:256-264)
* HER2K ``(alpha, z, b, beta, c)``            — kernels.her2k (kernels.py:267-281)

``c`` is a host complex128 F-order array updated in place (HERK/HER2K: lower
triangle only, Im(diag) := 0).  Operands are copied to the device, the
sm_100a kernel runs once (no host-side tiling: the device kernel tiles the
stored triangle itself), and ``c`` is copied back.  The default engine
("auto") is FP64 DMMA here -- elementwise FP64 rounding for arbitrary
operands, like the reference kernels; ``GpuPolicy(engine="int8")`` opts into
the INT8 emulation (FP64-width by default, normwise accurate).  ``ExecResult.seconds`` is the CUDA-event time of the kernel alone;
``n_tiles`` counts the 64 x 64 output tiles the kernel launched.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .hs_types import DimensionError, InputError
from .ledger import KernelKind, _kind_of
from .pipeline import GpuPolicy

TILE = 64
_ITEM = 16


@dataclass(frozen=True)
class ExecResult:
    seconds: float
    n_tiles: int
    bytes_touched: int


def _real(x, what):
    if isinstance(x, complex) and x.imag != 0:
        raise InputError(f"{what} must be real, got {x!r}")
    return float(np.real(x))


def _dev_matrix(m, dev):
    """Upload a host matrix; returns (tensor, ld) with the column-major data."""
    import torch

    a = np.asarray(m)
    if a.ndim != 2:
        raise DimensionError(f"expected a 2-D matrix, got ndim={a.ndim}")
    a = np.asfortranarray(a, dtype=np.complex128)
    t = torch.from_numpy(a.T).to(dev)  # row-major (cols, rows) == column-major (rows, cols)
    return t, max(1, a.shape[0])


def _stream_ptr(dev):
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _tiles(m, n, triangular):
    tm, tn = -(-m // TILE), -(-n // TILE)
    return tm * (tm + 1) // 2 if triangular else tm * tn


def _run_gpu(kind, operands, policy: GpuPolicy):
    import torch

    lib = _lib.load()
    dev = torch.device("cuda", policy.device)
    st = _stream_ptr(dev)
    if kind is KernelKind.HERK:
        alpha, a, beta, c = operands
        alpha, beta = _real(alpha, "herk alpha"), _real(beta, "herk beta")
        a = np.asarray(a)
        n = a.shape[1]
        if c.shape != (n, n):
            raise DimensionError(f"c has shape {c.shape}, expected {(n, n)}")
        da, lda = _dev_matrix(a, dev)
        dc, ldc = _dev_matrix(c, dev)
        call = lambda ctx: lib.hsb_zherk(ctx, st, n, a.shape[0], alpha, da.data_ptr(), lda, beta,
                                     dc.data_ptr(), ldc, 0)
        tiles = _tiles(n, n, True)
        touched = (c.size + 2 * a.size) * _ITEM
    elif kind is KernelKind.HER2K:
        alpha, z, b, beta, c = operands
        beta = _real(beta, "her2k beta")
        z, b = np.asarray(z), np.asarray(b)
        if z.shape != b.shape:
            raise DimensionError(f"z shape {z.shape} != b shape {b.shape}")
        n = z.shape[1]
        if c.shape != (n, n):
            raise DimensionError(f"c has shape {c.shape}, expected {(n, n)}")
        al = complex(alpha)
        dz, ldz = _dev_matrix(z, dev)
        db, ldb = _dev_matrix(b, dev)
        dc, ldc = _dev_matrix(c, dev)
        call = lambda ctx: lib.hsb_zher2k(ctx, st, n, z.shape[0], al.real, al.imag, dz.data_ptr(), ldz,
                                      db.data_ptr(), ldb, beta, dc.data_ptr(), ldc, 0)
        tiles = _tiles(n, n, True)
        touched = (c.size + 2 * (z.size + b.size)) * _ITEM
    else:
        alpha, opa, a, opb, b, beta, c = operands
        for op, name in ((opa, "a"), (opb, "b")):
            if op not in ("N", "T", "C"):
                raise InputError(f"unknown op {op!r} for operand {name}")
        a, b = np.asarray(a), np.asarray(b)
        m, ka = (a.shape if opa == "N" else a.shape[::-1])
        kb, n = (b.shape if opb == "N" else b.shape[::-1])
        if ka != kb:
            raise DimensionError(f"inner dimensions disagree: op(a) {(m, ka)} vs op(b) {(kb, n)}")
        if c.shape != (m, n):
            raise DimensionError(f"c has shape {c.shape}, expected {(m, n)}")
        al, be = complex(alpha), complex(beta)
        da, lda = _dev_matrix(a, dev)
        db, ldb = _dev_matrix(b, dev)
        dc, ldc = _dev_matrix(c, dev)
        call = lambda ctx: lib.hsb_zgemm(ctx, st, opa.encode(), opb.encode(), m, n, ka, al.real, al.imag,
                                     da.data_ptr(), lda, db.data_ptr(), ldb, be.real, be.imag,
                                     dc.data_ptr(), ldc, 0)
        tiles = _tiles(m, n, False)
        touched = (c.size + (m + n) * ka) * _ITEM
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with _lib.using(policy.device, policy.complex_mult, policy.engine, policy.int8_bits) as ctx:
        start.record()
        _lib.check(call(ctx), ctx)
        end.record()
    end.synchronize()
    host = dc.cpu().numpy().T  # column-major view
    c[...] = host
    return ExecResult(start.elapsed_time(end) * 1e-3, tiles, touched)


def run_partitioned(kind, operands: tuple, policy=None) -> ExecResult:
    """GPU ``run_partitioned``: same operand tuples and in-place semantics."""
    kind = _kind_of(kind)
    if kind not in (KernelKind.GEMM, KernelKind.HERK, KernelKind.HER2K):
        raise InputError(f"run_partitioned does not dispatch {kind!r}")
    policy = policy if isinstance(policy, GpuPolicy) else GpuPolicy()
    return _run_gpu(kind, operands, policy)
