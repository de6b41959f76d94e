"""Build the sm_100a shared library in-tree (travels to the GPU box with the repo).

    python -m paper_1503_06959_b200.build

nvcc -gencode arch=compute_100a,code=sm_100a; -fmad=false keeps every fp64
expression in the reference's operation order (numba emits no FMA; see
SURVEY.md section 0 "Numerics").
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libvidfeat_b200.so"
SOURCES = ["vf_capi.cu", "vf_match.cu", "vf_ransac.cu", "vf_format.cpp"]
DEPS = ["vf_capi.cu", "vf_kernels.cu", "vf_common.cuh", "vf_match.cu", "vf_temporal.cuh", "vf_format.cpp", "vf_ransac.cu",
        "vf_rng.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build vidfeat-b200")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    hdr = PKG.parent / "include" / "vidfeat_b200.h"
    return any((CSRC / d).stat().st_mtime > t for d in DEPS) or hdr.stat().st_mtime > t


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, *(str(CSRC / s) for s in SOURCES), "-o", str(tmp)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
