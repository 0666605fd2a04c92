"""The reference's acceptance criteria 3 and 4 (pkg/tests/test_acceptance.py:48-87)
on the B200 build, against fixtures the reference itself produced
(tests/golden/make_acceptance_golden.py):

* criterion 3 -- 100 randomized instances (1-6 atoms, 2-12 lm rows, 4-48 G
  vectors, nonhpd fractions 0 / 0.5 / 1) against the brute-force oracle
  h_reference / s_reference: the reference's tolerance is 1e-9; both engines
  are held to 1e-13 here;
* criterion 4 -- 50 HPD instances built normally and with force_nonhpd: the
  Cholesky and Hermitian-multiply routes agree (reference tolerance 1e-10)
  and each matches the reference's own build_hs output.

The CPU test pins the oracle restatement (oracle/brute.py) to the same fixtures.
"""

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1611_00606_b200 import Dims, GpuPolicy, ProblemSpec, build_hs, generate, rel_frob_error


def _fixtures():
    with np.load(GOLDEN / "acceptance.npz") as z:
        return {k: z[k] for k in z.files}


def _c3_instances(fx):
    for row in fx["c3_params"]:
        na, nl, ng, trial, frac = (int(row[0]), int(row[1]), int(row[2]), int(row[3]), float(row[4]))
        yield trial, generate(ProblemSpec(Dims(na, nl, ng), seed=trial, nonhpd_fraction=frac))


def test_oracle_matches_reference_acceptance_sweep():
    from oracle import brute

    fx = _fixtures()
    for trial, p in _c3_instances(fx):
        assert rel_frob_error(brute.h_brute(p), fx[f"c3_{trial}_h"]) < 1e-13
        assert rel_frob_error(brute.s_brute(p), fx[f"c3_{trial}_s"]) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["auto", "dmma"])
def test_criterion_3_oracle_equivalence_sweep(engine):
    fx = _fixtures()
    worst_h = worst_s = 0.0
    for trial, p in _c3_instances(fx):
        out = build_hs(p, GpuPolicy(engine=engine))
        eh = rel_frob_error(out.h.matrix, fx[f"c3_{trial}_h"])
        es = rel_frob_error(out.s.matrix, fx[f"c3_{trial}_s"])
        worst_h, worst_s = max(worst_h, eh), max(worst_s, es)
        assert eh <= 1e-13 and es <= 1e-13, (trial, eh, es)
    print(f"criterion 3 ({engine}): worst rel error H {worst_h:.2e}, S {worst_s:.2e}")


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["auto", "dmma"])
def test_criterion_4_cholesky_path_equivalence(engine):
    fx = _fixtures()
    worst = 0.0
    for trial, row in enumerate(fx["c4_params"]):
        na, nl, ng, seed = (int(x) for x in row[:4])
        p = generate(ProblemSpec(Dims(na, nl, ng), seed=seed, nonhpd_fraction=0.0))
        normal = build_hs(p, GpuPolicy(engine=engine))
        forced = build_hs(p, GpuPolicy(engine=engine), force_nonhpd=True)
        assert normal.split.nonhpd == 0 and forced.split.hpd == 0
        err = rel_frob_error(forced.h.matrix, normal.h.matrix)
        worst = max(worst, err)
        assert err <= 1e-13, (trial, err)
        assert rel_frob_error(normal.h.matrix, fx[f"c4_{trial}_h"]) <= 1e-13
        assert rel_frob_error(forced.h.matrix, fx[f"c4_{trial}_hf"]) <= 1e-13
    print(f"criterion 4 ({engine}): worst forced-vs-normal rel error {worst:.2e}")
