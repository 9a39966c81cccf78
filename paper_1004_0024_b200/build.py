"""Builds libisingb200.so (host C++ + sm_100a CUDA kernels) in-tree with nvcc.

    python -m paper_1004_0024_b200.build [--force]

-fmad=false: the reference forbids FP contraction (proj/src/CMakeLists.txt:23-29); the kernels
also spell every rounding step with explicit intrinsics.  -lineinfo keeps ncu's source page
mapped to the .cu files.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libisingb200.so"

SOURCES = ["host_model.cpp", "model_text.cpp", "batch.cpp", "coalesced.cpp", "capi.cpp", "kernels_generic.cu", "kernels_layered.cu", "kernels_strand.cu", "kernels_coalesced.cu"]
# ISING_NVCC_DEFINES: extra -D flags for timing experiments (profiles/), never set for the product build
NVCC_FLAGS = [*(["-DISING_STRAND_PROFILE"] if os.environ.get("ISING_STRAND_PROFILE") else []),
    *os.environ.get("ISING_NVCC_DEFINES", "").split(),
    "-std=c++17", "-O3", "-lineinfo", "-fmad=false",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-Wall,-Wextra,-fvisibility=hidden",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found: the CUDA extension cannot be built")
    return exe


FLAGS_STAMP = PKG / "build" / "flags.txt"  # the flags of the last build: other flags, other library


def needs_build() -> bool:
    if not LIB.exists():
        return True
    if not FLAGS_STAMP.exists() or FLAGS_STAMP.read_text() != " ".join(NVCC_FLAGS):
        return True
    newest = max(p.stat().st_mtime for p in list(CSRC.iterdir()) + [ROOT / "include" / "isingmc_b200.h"])
    return newest > LIB.stat().st_mtime


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objs = []
    for src in SOURCES:
        path = CSRC / src
        if not path.exists():
            continue
        obj = objdir / (path.stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, "-I", str(ROOT / "include"), "-I", str(CSRC), "-c", str(path), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}")
        (objdir / (path.stem + ".ptxas.log")).write_text(res.stderr)
        objs.append(str(obj))
    cmd = [nvcc, "-shared", "-o", str(LIB), *objs, "-gencode", "arch=compute_100a,code=sm_100a"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("link failed")
    FLAGS_STAMP.write_text(" ".join(NVCC_FLAGS))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
