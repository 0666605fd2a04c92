"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU.

The golden fixtures under tests/golden/ were produced by running the
reference package itself (tests/golden/make_golden.py); /root/reference is
not needed at test time.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (run on the GPU box)")


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN / "meta.json").read_text())


def golden_cases():
    meta = json.loads((GOLDEN / "meta.json").read_text())
    return sorted(k for k in meta if not k.startswith("_"))


def load_case(name):
    """(instance, fixture dict, meta) for a golden build case, digest-checked."""
    from paper_1611_00606_b200 import Dims, ProblemSpec, generate

    meta = json.loads((GOLDEN / "meta.json").read_text())[name]
    p = generate(ProblemSpec(Dims(*meta["dims"]), seed=meta["seed"], nonhpd_fraction=meta["nonhpd_fraction"]))
    with np.load(GOLDEN / f"build_{name}.npz") as z:
        fx = {k: z[k] for k in z.files}
    return p, fx, meta
