"""HSM1 instance I/O (paper_1611_00606_b200/storage.py) against the reference
format: files written by the reference's own storage code
(tests/golden/hsm_tiny, made by tests/golden/make_hsm_golden.py) must load
bit-exactly and re-write byte-identically; the error cases follow
/root/reference/pkg/tests/test_storage.py.  The GPU-backed run_instance_dir
is checked against the reference's H.hsm / S.hsm (north star 1e-10)."""

import json
import shutil
import struct

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1611_00606_b200 import Dims, ProblemSpec, generate, rel_frob_error
from paper_1611_00606_b200.storage import (
    StorageError, load_instance, read_matrix, read_vector, run_instance_dir, save_instance, write_matrix,
    write_vector,
)

TINY = GOLDEN / "hsm_tiny"


def _cm(rng, r, c):
    return np.asfortranarray(rng.standard_normal((r, c)) + 1j * rng.standard_normal((r, c)))


def test_reads_reference_written_instance_and_rewrites_identically(tmp_path):
    inst = load_instance(TINY, pinned=False)
    assert (inst.dims.n_atoms, inst.dims.n_l, inst.dims.n_g) == (2, 4, 6)
    manifest = json.loads((TINY / "manifest.json").read_text())
    save_instance(inst, tmp_path, seed=manifest["seed"], nonhpd_fraction=manifest["nonhpd_fraction"])
    for f in sorted(TINY.iterdir()):
        if f.is_file():
            assert (tmp_path / f.name).read_bytes() == f.read_bytes(), f.name
    # and the generator reproduces the same bytes (instances.generate is hsgen-identical)
    p = generate(ProblemSpec(Dims(2, 4, 6), seed=21, nonhpd_fraction=0.5))
    for name in ("a_blocks", "b_blocks", "t_aa", "t_ab", "t_bb", "u_norms"):
        for x, y in zip(getattr(p, name), getattr(inst, name)):
            assert x.tobytes() == y.tobytes()
            assert y.flags.f_contiguous


def test_matrix_roundtrip_and_header(tmp_path):
    rng = np.random.default_rng(1)
    for shape in [(1, 1), (3, 5), (7, 2), (0, 3)]:
        m = _cm(rng, *shape)
        write_matrix(tmp_path / "m.hsm", m)
        back = read_matrix(tmp_path / "m.hsm")
        assert back.shape == m.shape and back.tobytes() == m.tobytes() and back.flags.f_contiguous
    write_matrix(tmp_path / "h.hsm", np.array([[1 + 2j, 3 + 4j]]))
    data = (tmp_path / "h.hsm").read_bytes()
    assert len(data) == 25 + 32
    assert struct.unpack_from("<4sIBQQ", data) == (b"HSM1", 1, 1, 1, 2)
    assert struct.unpack_from("<4d", data, 25) == (1.0, 2.0, 3.0, 4.0)


def test_matrix_and_vector_errors(tmp_path):
    (tmp_path / "short.hsm").write_bytes(b"HSM1\x01")
    with pytest.raises(StorageError, match="short.hsm"):
        read_matrix(tmp_path / "short.hsm")
    (tmp_path / "bad.hsm").write_bytes(b"XXXX" + b"\x00" * 30)
    with pytest.raises(StorageError, match="magic"):
        read_matrix(tmp_path / "bad.hsm")
    write_matrix(tmp_path / "t.hsm", np.eye(3, dtype=complex))
    (tmp_path / "t.hsm").write_bytes((tmp_path / "t.hsm").read_bytes()[:-8])
    with pytest.raises(StorageError, match="payload"):
        read_matrix(tmp_path / "t.hsm")
    with pytest.raises(StorageError):
        write_matrix(tmp_path / "v.hsm", np.zeros(3))
    write_vector(tmp_path / "u.f64", np.arange(3.0))
    assert read_vector(tmp_path / "u.f64").tolist() == [0.0, 1.0, 2.0]
    (tmp_path / "u.f64").write_bytes(b"\x00" * 7)
    with pytest.raises(StorageError, match="multiple of 8"):
        read_vector(tmp_path / "u.f64")


def test_instance_directory_errors(tmp_path):
    with pytest.raises(StorageError, match="manifest"):
        load_instance(tmp_path, pinned=False)
    d = tmp_path / "i"
    shutil.copytree(TINY, d)
    (d / "t_aa_0002.hsm").unlink()
    with pytest.raises(StorageError, match="t_aa_0002.hsm"):
        load_instance(d, pinned=False)
    shutil.copy(TINY / "t_aa_0002.hsm", d)
    write_matrix(d / "a_0001.hsm", np.zeros((5, 5), dtype=complex))
    with pytest.raises(StorageError, match="a_0001.hsm"):
        load_instance(d, pinned=False)
    shutil.copy(TINY / "a_0001.hsm", d)
    m = json.loads((d / "manifest.json").read_text())
    del m["dims"]
    (d / "manifest.json").write_text(json.dumps(m))
    with pytest.raises(StorageError, match="malformed"):
        load_instance(d, pinned=False)


@pytest.mark.gpu
def test_run_instance_dir_matches_reference_outputs(tmp_path):
    d = tmp_path / "i"
    shutil.copytree(TINY, d)
    report = run_instance_dir(d)
    h, s = read_matrix(d / "H.hsm"), read_matrix(d / "S.hsm")
    assert rel_frob_error(h, read_matrix(TINY / "reference_outputs" / "H.hsm")) < 1e-10
    assert rel_frob_error(s, read_matrix(TINY / "reference_outputs" / "S.hsm")) < 1e-10
    assert report["split"]["hpd"] + report["split"]["nonhpd"] == 2
    assert json.loads((d / "report.json").read_text())["total_flops"] == report["total_flops"]
    inst = load_instance(d, pinned=True)  # page-locked blocks (direct DMA path)
    assert inst.a_blocks[0].flags.f_contiguous
    for name in ("a_blocks", "t_ab", "u_norms"):
        for x, y in zip(getattr(inst, name), getattr(load_instance(TINY, pinned=False), name)):
            assert x.tobytes() == y.tobytes()
