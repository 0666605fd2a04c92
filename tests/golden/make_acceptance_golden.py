"""Golden fixtures for the reference's acceptance criteria 3 and 4, made by
running the reference itself (pkg/tests/test_acceptance.py:48-87).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_acceptance_golden.py

Criterion 3: 100 randomized instances (dims drawn by numpy default_rng(2024)
exactly as the reference's sweep draws them, seed = trial, nonhpd fraction
cycling 0, 0.5, 1) -> the brute-force oracle h_reference / s_reference.
Criterion 4: 50 HPD instances (default_rng(77), seed 1000 + trial) ->
build_hs with and without force_nonhpd.  Stored as acceptance.npz with the
instance parameters; tests/test_gpu_acceptance.py regenerates each instance
with the repo's bit-identical generator and checks the B200 build.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from hsgen.builder import build_hs  # noqa: E402
from hsgen.matcore import Dims  # noqa: E402
from hsgen.probgen import ProblemSpec, generate  # noqa: E402
from hsgen.reference import h_reference, s_reference  # noqa: E402

HERE = Path(__file__).resolve().parent


def main():
    out = {}
    rng = np.random.default_rng(2024)
    fractions = [0.0, 0.5, 1.0]
    c3 = []
    for trial in range(100):
        dims = (int(rng.integers(1, 7)), int(rng.integers(2, 13)), int(rng.integers(4, 49)))
        frac = fractions[trial % 3]
        p = generate(ProblemSpec(Dims(*dims), seed=trial, nonhpd_fraction=frac))
        out[f"c3_{trial}_h"] = h_reference(p).matrix
        out[f"c3_{trial}_s"] = s_reference(p).matrix
        c3.append((*dims, trial, frac))
    out["c3_params"] = np.array(c3, dtype=np.float64)
    rng = np.random.default_rng(77)
    c4 = []
    for trial in range(50):
        dims = (int(rng.integers(1, 5)), int(rng.integers(2, 9)), int(rng.integers(4, 25)))
        p = generate(ProblemSpec(Dims(*dims), seed=1000 + trial, nonhpd_fraction=0.0))
        normal, forced = build_hs(p), build_hs(p, force_nonhpd=True)
        out[f"c4_{trial}_h"] = normal.h.matrix
        out[f"c4_{trial}_hf"] = forced.h.matrix
        c4.append((*dims, 1000 + trial, normal.split.nonhpd, forced.split.hpd))
    out["c4_params"] = np.array(c4, dtype=np.float64)
    np.savez_compressed(HERE / "acceptance.npz", **out)
    print("wrote", HERE / "acceptance.npz")


if __name__ == "__main__":
    main()
