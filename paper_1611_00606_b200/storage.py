"""HSM1 instance I/O feeding the B200 build directly.

Same on-disk formats and error behaviour as ``hsgen.storage``
(/root/reference/pkg/src/hsgen/storage.py):

* ``.hsm`` matrix: 25-byte little-endian header ``"HSM1"``, version u32 = 1,
  dtype u8 = 1 (complex128), rows u64, cols u64, then the column-major
  ``<c16`` payload (storage.py:16-55);
* ``.f64`` vector: raw ``<f8`` (storage.py:58-65);
* ``manifest.json``: ``dims``, ``seed``, ``nonhpd_fraction`` and per-field file
  lists ``a, b, t_aa, t_ab, t_bb, u`` (storage.py:70-104), checked on load
  against the dims (storage.py:107-167).

The difference is where the bytes land: ``load_instance(..., pinned=True)``
reads every block straight from the file into page-locked host memory (one
``readinto`` per block, no intermediate copy), so ``build_hs`` DMAs it to the
device without staging.  ``run_instance_dir`` is the GPU-backed counterpart
of ``hsgen run`` (cli.py:147-183): load, build, write ``H.hsm`` / ``S.hsm``
and the same ``report.json`` schema.
"""

from __future__ import annotations

import json
import struct
import time
from pathlib import Path

import numpy as np

from .hs_types import Dims, reference_module
from .instances import ProblemInstance

MAGIC = b"HSM1"
HEADER = struct.Struct("<4sIBQQ")  # magic, version, dtype tag, rows, cols: 25 bytes
VERSION = 1
DTYPE_COMPLEX128 = 1
MANIFEST_NAME = "manifest.json"
BLOCK_FIELDS = ("a", "b", "t_aa", "t_ab", "t_bb")
_INSTANCE_ATTR = {"a": "a_blocks", "b": "b_blocks", "t_aa": "t_aa", "t_ab": "t_ab", "t_bb": "t_bb"}


_REF_STORAGE = reference_module("storage")
if _REF_STORAGE is not None:
    StorageError = _REF_STORAGE.StorageError  # the reference's class (storage.py:23-24)
else:
    class StorageError(ValueError):
        """A file is missing, truncated, or inconsistent with its manifest (storage.py:23-24)."""


def _empty_matrix(rows: int, cols: int, pinned: bool) -> np.ndarray:
    if pinned:
        import torch

        return torch.empty((cols, rows), dtype=torch.complex128, pin_memory=True).numpy().T
    return np.empty((rows, cols), dtype=np.complex128, order="F")


def _read_header(fh, path) -> tuple[int, int]:
    head = fh.read(HEADER.size)
    if len(head) < HEADER.size:
        raise StorageError(f"{path}: file shorter than the 25-byte header")
    magic, version, dtype, rows, cols = HEADER.unpack(head)
    if magic != MAGIC:
        raise StorageError(f"{path}: bad magic {magic!r}")
    if version != VERSION or dtype != DTYPE_COMPLEX128:
        raise StorageError(f"{path}: unsupported version/dtype {version}/{dtype}")
    return rows, cols


def read_matrix(path, pinned: bool = False, expect_shape=None) -> np.ndarray:
    """Read an HSM1 matrix (F-order complex128); optionally into pinned memory."""
    path = Path(path)
    size = path.stat().st_size
    with open(path, "rb") as fh:
        rows, cols = _read_header(fh, path)
        payload = size - HEADER.size
        if payload != 16 * rows * cols:
            raise StorageError(f"{path}: payload is {payload} bytes, expected {16 * rows * cols}")
        if expect_shape is not None and (rows, cols) != tuple(expect_shape):
            raise StorageError(f"{path}: shape {(rows, cols)} does not match manifest {tuple(expect_shape)}")
        out = _empty_matrix(rows, cols, pinned)
        if rows * cols:
            view = memoryview(out.T.reshape(-1).view(np.uint8))  # F-order bytes of `out`
            got = fh.readinto(view)
            if got != 16 * rows * cols:
                raise StorageError(f"{path}: short read ({got} of {16 * rows * cols} bytes)")
    return out


def write_matrix(path, m) -> None:
    m = np.asarray(m)
    if m.ndim != 2:
        raise StorageError(f"{path}: only 2-D matrices can be written")
    m = np.asfortranarray(m, dtype=np.complex128)
    with open(path, "wb") as fh:
        fh.write(HEADER.pack(MAGIC, VERSION, DTYPE_COMPLEX128, m.shape[0], m.shape[1]))
        if m.size:
            fh.write(memoryview(m.T.reshape(-1).view(np.uint8)))  # no byte-order copy on little-endian hosts


def read_vector(path, pinned: bool = False) -> np.ndarray:
    path = Path(path)
    data = path.read_bytes()
    if len(data) % 8:
        raise StorageError(f"{path}: length {len(data)} is not a multiple of 8")
    v = np.frombuffer(data, dtype="<f8").astype(np.float64)
    if pinned:
        import torch

        out = torch.empty(v.shape, dtype=torch.float64, pin_memory=True).numpy()
        out[...] = v
        return out
    return v


def write_vector(path, v) -> None:
    v = np.asarray(v, dtype=np.float64)
    if v.ndim != 1:
        raise StorageError(f"{path}: only 1-D vectors can be written")
    Path(path).write_bytes(v.astype("<f8", copy=False).tobytes())


def save_instance(p, outdir, seed: int = 0, nonhpd_fraction: float = 0.0) -> dict:
    """Write the per-atom block files and the manifest (storage.py:73-104); returns the manifest."""
    outdir = Path(outdir)
    outdir.mkdir(parents=True, exist_ok=True)
    files: dict[str, list[str]] = {}
    for field in BLOCK_FIELDS:
        files[field] = []
        for a, blk in enumerate(getattr(p, _INSTANCE_ATTR[field])):
            name = f"{field}_{a + 1:04d}.hsm"
            write_matrix(outdir / name, blk)
            files[field].append(name)
    files["u"] = []
    for a, u in enumerate(p.u_norms):
        name = f"u_{a + 1:04d}.f64"
        write_vector(outdir / name, u)
        files["u"].append(name)
    manifest = {"dims": {"n_atoms": p.dims.n_atoms, "n_l": p.dims.n_l, "n_g": p.dims.n_g},
                "seed": seed, "nonhpd_fraction": nonhpd_fraction, "files": files}
    (outdir / MANIFEST_NAME).write_text(json.dumps(manifest, indent=2, sort_keys=True) + "\n")
    return manifest


def load_instance(indir, pinned: bool = True) -> ProblemInstance:
    """Read an instance directory, checking every file against the manifest
    (storage.py:107-167).  With ``pinned`` the blocks are page-locked, ready
    for direct DMA by ``build_hs``."""
    indir = Path(indir)
    mpath = indir / MANIFEST_NAME
    if not mpath.is_file():
        raise StorageError(f"{mpath}: manifest not found")
    try:
        manifest = json.loads(mpath.read_text())
        dims = Dims(**manifest["dims"])
        files = manifest["files"]
    except (json.JSONDecodeError, KeyError, TypeError, ValueError) as exc:
        raise StorageError(f"{mpath}: malformed manifest ({exc})") from exc
    shapes = {"a": (dims.n_l, dims.n_g), "b": (dims.n_l, dims.n_g), "t_aa": (dims.n_l, dims.n_l),
              "t_ab": (dims.n_l, dims.n_l), "t_bb": (dims.n_l, dims.n_l)}
    inst = ProblemInstance(dims)
    for field in BLOCK_FIELDS:
        names = files.get(field, [])
        if len(names) != dims.n_atoms:
            raise StorageError(f"{mpath}: {len(names)} {field} files listed, expected {dims.n_atoms}")
        blocks = getattr(inst, _INSTANCE_ATTR[field])
        for name in names:
            path = indir / name
            if not path.is_file():
                raise StorageError(f"{path}: referenced by manifest but missing")
            blocks.append(read_matrix(path, pinned=pinned, expect_shape=shapes[field]))
    unames = files.get("u", [])
    if len(unames) != dims.n_atoms:
        raise StorageError(f"{mpath}: {len(unames)} u files listed, expected {dims.n_atoms}")
    for name in unames:
        path = indir / name
        if not path.is_file():
            raise StorageError(f"{path}: referenced by manifest but missing")
        u = read_vector(path, pinned=pinned)
        if u.shape != (dims.n_l,):
            raise StorageError(f"{path}: length {u.shape[0]} does not match manifest {dims.n_l}")
        inst.u_norms.append(u)
    return inst


def run_instance_dir(indir, policy=None, report_path=None) -> dict:
    """GPU-backed ``hsgen run`` (cli.py:147-183): load the instance into pinned
    memory, build H and S on the B200, write ``H.hsm``, ``S.hsm`` and the
    report (same JSON schema; the efficiency denominator is the measured B200
    FP64 DMMA peak instead of the paper's 2 x K20x + CPU peak)."""
    from .pipeline import _policy, build_hs
    from .report import B200_FP64_PEAK_GFLOPS, summarize

    indir = Path(indir)
    inst = load_instance(indir, pinned=True)
    pol = _policy(policy)
    t0 = time.perf_counter()
    out = build_hs(inst, pol)
    wall = time.perf_counter() - t0
    write_matrix(indir / "H.hsm", out.h.matrix)
    write_matrix(indir / "S.hsm", out.s.matrix)
    sections = summarize(out.ledger, B200_FP64_PEAK_GFLOPS)
    report = {
        "policy": {"device": pol.device, "engine": pol.engine, "fused": pol.fused},
        "split": {"hpd": out.split.hpd, "nonhpd": out.split.nonhpd},
        "peak_gflops": B200_FP64_PEAK_GFLOPS,
        "total_seconds": wall,
        "total_flops": out.ledger.total_flops(),
        "sections": [{"section": r.section, "seconds": r.seconds, "flops": r.flops,
                      "gflops_per_s": r.gflops_per_s, "efficiency": r.efficiency} for r in sections],
    }
    rpath = Path(report_path) if report_path else indir / "report.json"
    rpath.write_text(json.dumps(report, indent=2) + "\n")
    return report
