"""Boundary fidelity with the reference package installed (CPU, no GPU).

When ``hsgen`` is importable the drop-in raises the reference's own
exception classes (matcore.py:16-25, storage.py:23-24) and returns its
``BuildOutput`` (builder.py:51-62), so ``hsgen.cli.cmd_run``'s
``except InvariantError`` (cli.py:161) maps a bad instance to exit code 3.
Each case runs in a subprocess with the reference on PYTHONPATH, as a user's
environment would have it; skipped where /root/reference is absent.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import ROOT

REF_SRC = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF_SRC.is_dir(), reason="reference package not present")


def _run(code: str, tmp_path) -> subprocess.CompletedProcess:
    env = dict(os.environ, PYTHONPATH=f"{ROOT}{os.pathsep}{REF_SRC}")
    env.pop("HSB200_STANDALONE", None)
    return subprocess.run([sys.executable, "-c", code], cwd=tmp_path, env=env, capture_output=True, text=True,
                          timeout=300)


def test_exception_classes_are_the_references(tmp_path):
    r = _run("""
import hsgen.matcore as m, hsgen.storage as st
import paper_1611_00606_b200 as d
from paper_1611_00606_b200 import storage, _lib
assert d.InvariantError is m.InvariantError and d.InputError is m.InputError
assert d.DimensionError is m.DimensionError and storage.StorageError is st.StorageError
from paper_1611_00606_b200 import instances, pipeline
assert instances.InvariantError is m.InvariantError and pipeline.InvariantError is m.InvariantError
assert _lib.InvariantError is m.InvariantError
# the ABI status -> exception mapping raises the reference's classes too
for status, cls in ((_lib.HSB_ERR_INVARIANT, m.InvariantError), (_lib.HSB_ERR_DIMENSION, m.DimensionError),
                    (_lib.HSB_ERR_INPUT, m.InputError)):
    try:
        _lib.check(status, None)
    except cls:
        pass
    else:
        raise SystemExit("no exception for status %d" % status)
print("ok")
""", tmp_path)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr


def test_cli_run_maps_drop_in_invariant_error_to_exit_3(tmp_path):
    # hsgen.cli.cmd_run with the drop-in's build_hs: an instance whose T_AB
    # block has the wrong shape must exit EXIT_INVARIANT (3), not traceback
    r = _run("""
import numpy as np
import hsgen.cli as cli
from hsgen.probgen import ProblemSpec, generate
from hsgen.matcore import Dims
import paper_1611_00606_b200 as d
p = generate(ProblemSpec(Dims(2, 3, 5), seed=1))
p.t_ab[1] = np.zeros((2, 2), dtype=complex, order="F")
cli.load_instance = lambda _dir: p
cli.build_hs = d.build_hs
rc = cli.main(["run", "--in", "."])
print("rc", rc)
""", tmp_path)
    assert "rc 3" in r.stdout, (r.stdout, r.stderr)
    assert "instance invariant violated" in r.stderr


def test_validation_order_matches_reference_when_several_fields_are_bad(tmp_path):
    # non-finite A together with a non-Hermitian T_AA: the reference reports
    # a_blocks first (probgen.py:140-168); the drop-in's host validation too
    r = _run("""
import numpy as np
from hsgen.probgen import ProblemSpec, generate, validate_instance as ref_validate
from hsgen.matcore import Dims, InvariantError
from paper_1611_00606_b200 import validate_instance
p = generate(ProblemSpec(Dims(2, 3, 5), seed=2))
p.a_blocks[1][0, 0] = np.nan
p.b_blocks[0][1, 1] = np.inf
p.t_aa[0][0, 1] += 1.0
msgs = []
for fn in (ref_validate, validate_instance):
    try:
        fn(p)
    except InvariantError as e:
        msgs.append(str(e))
assert len(msgs) == 2 and msgs[0].split()[0] == msgs[1].split()[0] == "a_blocks[1]", msgs
print("ok")
""", tmp_path)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout, r.stderr)
