"""The C-ABI library loads and exports every symbol include/hsb200.h declares
(no compute calls: this runs without a GPU)."""

import ctypes
import re

import pytest

from conftest import ROOT
from paper_1611_00606_b200 import _lib


def _declared():
    text = (ROOT / "include" / "hsb200.h").read_text()
    return re.findall(r"HSB_API\s+[\w\s\*]*?\b(hsb_\w+)\s*\(", text)


def test_header_declares_the_boundary():
    names = set(_declared())
    assert {"hsb_ctx_create", "hsb_ctx_destroy", "hsb_last_error", "hsb_zherk", "hsb_zher2k", "hsb_zgemm",
            "hsb_hermitian_mirror", "hsb_build_hs", "hsb_abi_version"} <= names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_loader_and_abi_version():
    lib = _lib.load()
    assert lib.hsb_abi_version() == _lib.ABI_VERSION == 8


def test_binding_struct_layout_matches_header():
    # 3*8 + 2*4 + 6 pointers + 6 pointers
    assert ctypes.sizeof(_lib.HsbProblem) == 32 + 12 * 8
    assert ctypes.sizeof(_lib.HsbOutput) == 8 + 8 + 10 * 8  # h, s, peer, s_ready, 4 events, 2 flags
    assert ctypes.sizeof(_lib.HsbPeerOut) == 8 + 8 + 8 + 16
    assert ctypes.sizeof(_lib.HsbTimings) == 13 * 8 + 16 + 2 * 8


def test_kernels_are_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_int8_crt_table_matches_restatement():
    # the table the device reconstructs with (csrc/ozaki.cu oz_crt_table,
    # exported host-side) equals the Python restatement bit for bit
    import numpy as np

    from paper_1611_00606_b200.engine import MODULI, crt_weights

    lib = _lib.load()
    for n_mod in range(11, len(MODULI) + 1):
        w = np.zeros((2, n_mod, 2))
        m = ctypes.c_double()
        assert lib.hsb_oz_crt_table(n_mod, w.ctypes.data, ctypes.byref(m)) == 0
        want, want_m = crt_weights(n_mod)
        assert w.tolist() == [[list(x) for x in part] for part in want]
        assert m.value == want_m
    assert lib.hsb_oz_crt_table(21, w.ctypes.data, ctypes.byref(m)) != 0
