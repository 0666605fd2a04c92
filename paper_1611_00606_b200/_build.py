"""Build libhsb200.so in-tree with nvcc for sm_100a (no torch involvement).

    python -m paper_1611_00606_b200._build [--force]

The shared library is the C-ABI of include/hsb200.h.  It is written next to
this file so it travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libhsb200.so"
SOURCES = ["zrk_kernel.cu", "zrk3m_kernel.cu", "aux_kernels.cu", "staging.cu", "match_kernel.cu", "ozaki.cu", "contract.cu", "hsb_api.cu"]
HEADERS = ["zrk.cuh", "ptx.cuh", "ozaki.cuh", "ozaki_res.cuh", "host_ctx.cuh", "aux_kernels.cuh", "staging.cuh", "match.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-warn-spills", "-Xcompiler", "-fopenmp",
    f"-I{ROOT / 'include'}",
]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; cannot build libhsb200.so")
    return cand


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "hsb200.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    objs = [str(objdir / (Path(src).stem + ".o")) for src in SOURCES]

    def compile_one(src_obj):
        src, obj = src_obj
        cmd = [nvcc(), *NVCC_FLAGS, "-c", str(CSRC / src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)

    # translation units are independent: compile them concurrently
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as pool:
        list(pool.map(compile_one, zip(SOURCES, objs)))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fopenmp", *objs, "-lgomp", "-o", str(tmp)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
