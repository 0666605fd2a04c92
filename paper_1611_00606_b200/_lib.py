"""ctypes binding of libhsb200.so (the C ABI declared in include/hsb200.h).

There is no fallback: if the shared library is missing or cannot be loaded
the import of anything that needs it raises ``RuntimeError``.  Build it with
``python -m paper_1611_00606_b200._build`` (``__graft_entry__.build()``).
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import threading
from pathlib import Path

from .hs_types import DimensionError, InputError, InvariantError

LIB_PATH = Path(os.environ.get("HSB200_LIB", Path(__file__).resolve().parent / "libhsb200.so"))

HSB_OK, HSB_ERR_DIMENSION, HSB_ERR_INPUT, HSB_ERR_INVARIANT = 0, 1, 2, 3
HSB_ERR_CUDA, HSB_ERR_UNSUPPORTED, HSB_ERR_NOMEM = 4, 5, 6

HSB_LOWER_ONLY = 0x1
HSB_MIRROR = 0x2
HSB_LOC_HOST = 0
HSB_LOC_DEVICE = 1
HSB_OPT_FORCE_NONHPD = 0x1
HSB_OPT_UNFUSED = 0x2
HSB_OPT_VALIDATE = 0x4
HSB_OPT_FULL_D2H = 0x8
HSB_OPT_LOWER_ONLY = 0x10
HSB_CPLX_4M = 0
HSB_CPLX_3M = 1
COMPLEX_MULT = {"4m": HSB_CPLX_4M, "3m": HSB_CPLX_3M}
HSB_ENGINE_DMMA = 0
HSB_ENGINE_INT8 = 1
HSB_ENGINE_AUTO = 2
ENGINES = {"dmma": HSB_ENGINE_DMMA, "int8": HSB_ENGINE_INT8, "auto": HSB_ENGINE_AUTO}
ABI_VERSION = 8

_P = ctypes.c_void_p
_DPP = ctypes.POINTER(ctypes.c_void_p)


class HsbProblem(ctypes.Structure):
    _fields_ = [
        ("n_atoms", ctypes.c_int64), ("n_l", ctypes.c_int64), ("n_g", ctypes.c_int64),
        ("location", ctypes.c_int32), ("reserved", ctypes.c_int32),
        ("a_blocks", _DPP), ("b_blocks", _DPP), ("t_aa", _DPP), ("t_ab", _DPP),
        ("t_bb", _DPP), ("u_norms", _DPP),
        ("a_stack", _P), ("b_stack", _P), ("t_aa_dev", _P), ("t_ab_dev", _P),
        ("t_bb_dev", _P), ("u_dev", _P),
    ]


class HsbPeerOut(ctypes.Structure):
    _fields_ = [("n_ranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("cols_per_rank", ctypes.c_int64),
                ("ld", ctypes.c_int64), ("h_slots", _P), ("s_slots", _P)]


class HsbOutput(ctypes.Structure):
    _fields_ = [("location", ctypes.c_int32), ("reserved", ctypes.c_int32), ("ld", ctypes.c_int64),
                ("h", _P), ("s", _P), ("peer", ctypes.POINTER(HsbPeerOut)), ("s_ready", _P),
                ("h2d_after", _P), ("h2d_done", _P), ("compute_after", _P), ("compute_done", _P),
                ("order_in", ctypes.POINTER(ctypes.c_int32)), ("order_out", ctypes.POINTER(ctypes.c_int32))]


class HsbTimings(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("loop1", "loop2", "unorm", "s1", "s2", "h1", "h2", "h3", "h2d", "d2h", "total",
                 "s_core", "h_core")] + [
        ("n_hpd", ctypes.c_int32), ("n_nonhpd", ctypes.c_int32), ("launches", ctypes.c_int32),
        ("reserved", ctypes.c_int32), ("h2d_bytes", ctypes.c_double), ("d2h_bytes", ctypes.c_double)]


class HsbPhys(ctypes.Structure):
    _fields_ = [("n_atoms", ctypes.c_int64), ("n_g", ctypes.c_int64), ("lmax", ctypes.c_int32),
                ("n_types", ctypes.c_int32), ("gvec", _P), ("tau", _P), ("type_of", _P), ("rmt", _P),
                ("radial", _P), ("kpt", ctypes.c_double * 3), ("recip", ctypes.c_double * 9),
                ("omega", ctypes.c_double)]


_lib = None
_lock = threading.Lock()
_ctxs: dict[tuple[int, int], ctypes.c_void_p] = {}
_ctx_locks: dict[tuple[int, int], threading.Lock] = {}


def load():
    """Load libhsb200.so once and declare the prototypes."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: the B200 kernels are not built "
                "(run `python -m paper_1611_00606_b200._build`); there is no CPU fallback")
        lib = ctypes.CDLL(os.fspath(LIB_PATH))
        i32, i64, dbl, u32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_uint32
        ch = ctypes.c_char
        sig = {
            "hsb_abi_version": (i32, []),
            "hsb_ctx_create": (i32, [i32, ctypes.POINTER(ctypes.c_void_p)]),
            "hsb_ctx_destroy": (None, [_P]),
            "hsb_last_error": (ctypes.c_char_p, [_P]),
            "hsb_ctx_trim": (i32, [_P]),
            "hsb_ctx_set_complex_mult": (i32, [_P, i32]),
            "hsb_ctx_set_engine": (i32, [_P, i32, i32]),
            "hsb_oz_crt_table": (i32, [i32, _P, _P]),
            "hsb_ipc_handle": (i32, [_P, _P, ctypes.c_char_p]),
            "hsb_ipc_open": (i32, [_P, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
            "hsb_ipc_close": (i32, [_P, _P]),
            "hsb_zherk": (i32, [_P, _P, i64, i64, dbl, _P, i64, dbl, _P, i64, u32]),
            "hsb_zher2k": (i32, [_P, _P, i64, i64, dbl, dbl, _P, i64, _P, i64, dbl, _P, i64, u32]),
            "hsb_zgemm": (i32, [_P, _P, ch, ch, i64, i64, i64, dbl, dbl, _P, i64, _P, i64, dbl, dbl,
                                _P, i64, u32]),
            "hsb_hermitian_mirror": (i32, [_P, _P, i64, _P, i64]),
            "hsb_sum_slots": (i32, [_P, _P, _P, i32, i64, i64, _P]),
            "hsb_match_coeffs": (i32, [_P, _P, ctypes.POINTER(HsbPhys), _P, _P, i64]),
            "hsb_build_hs_physical": (i32, [_P, _P, ctypes.POINTER(HsbPhys), ctypes.POINTER(HsbProblem), u32,
                                            ctypes.POINTER(HsbOutput), ctypes.POINTER(HsbTimings),
                                            ctypes.POINTER(ctypes.c_int32)]),
            "hsb_build_hs": (i32, [_P, _P, ctypes.POINTER(HsbProblem), u32, ctypes.POINTER(HsbOutput),
                                   ctypes.POINTER(HsbTimings), ctypes.POINTER(ctypes.c_int32)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.hsb_abi_version() != ABI_VERSION:
            raise RuntimeError("libhsb200.so ABI version mismatch; rebuild it")
        _lib = lib
        return lib


def check(status: int, ctx) -> None:
    """Map an hsb_status onto the reference's exception classes."""
    if status == HSB_OK:
        return
    msg = (load().hsb_last_error(ctx) or b"").decode(errors="replace")
    if status == HSB_ERR_DIMENSION:
        raise DimensionError(msg)
    if status == HSB_ERR_INPUT:
        raise InputError(msg)
    if status == HSB_ERR_INVARIANT:
        raise InvariantError(msg)
    raise RuntimeError(f"libhsb200 error {status}: {msg}")


def context(device: int = 0, complex_mult: str | None = None, engine: str | None = None, int8_bits: int = 0,
            slot: int = 0):
    """Process-wide context ``slot`` of ``device`` (created on first use).

    Each context owns its device workspace, copy stream and pinned staging, so
    builds on different slots (and streams) may run concurrently: the k-point
    pipeline (pipeline.build_hs_kpoints) overlaps one k-point's transfers
    with another's kernels this way.

    ``complex_mult`` ("3m" | "4m") selects the real-product form of the
    complex contractions for the calls that follow (hsb_ctx_set_complex_mult);
    ``engine`` ("auto" | "dmma" | "int8") the engine of the triangle
    contractions (hsb_ctx_set_engine; ``int8_bits`` 0 = default 53).  Settings
    are sticky per context: callers that change them use ``using`` so no other
    thread's call runs between the settings and the call.
    """
    lib = load()
    if complex_mult is not None and complex_mult not in COMPLEX_MULT:
        raise InputError(f"complex_mult must be one of {sorted(COMPLEX_MULT)}, got {complex_mult!r}")
    if engine is not None and engine not in ENGINES:
        raise InputError(f"engine must be one of {sorted(ENGINES)}, got {engine!r}")
    with _lock:
        ctx = _ctxs.get((device, slot))
        if ctx is None:
            out = ctypes.c_void_p()
            check(lib.hsb_ctx_create(device, ctypes.byref(out)), None)
            ctx = out
            _ctxs[(device, slot)] = ctx
            _ctx_locks[(device, slot)] = threading.Lock()
        if complex_mult is not None:
            check(lib.hsb_ctx_set_complex_mult(ctx, COMPLEX_MULT[complex_mult]), ctx)
        if engine is not None:
            check(lib.hsb_ctx_set_engine(ctx, ENGINES[engine], int(int8_bits)), ctx)
        return ctx


@contextlib.contextmanager
def using(device: int = 0, complex_mult: str | None = None, engine: str | None = None, int8_bits: int = 0,
          slot: int = 0):
    """``context(...)`` held for the duration of a ``with`` block: the settings
    and the calls inside apply together even when other threads use the same
    context with other settings (ctypes releases the GIL during the calls; the
    library serialises the calls themselves per context)."""
    context(device, slot=slot)  # create it and its lock
    with _ctx_locks[(device, slot)]:
        yield context(device, complex_mult, engine, int8_bits, slot)


def release_all() -> None:
    lib = load()
    with _lock:
        for ctx in _ctxs.values():
            lib.hsb_ctx_destroy(ctx)
        _ctxs.clear()


def trim_all(device: int | None = None) -> None:
    """Release the cached device workspace of every context (of ``device``);
    the next call on a context re-allocates what it needs."""
    lib = load()
    with _lock:
        for (dev, _slot), ctx in _ctxs.items():
            if device is None or dev == device:
                check(lib.hsb_ctx_trim(ctx), ctx)
