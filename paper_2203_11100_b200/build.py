"""Builds libswb200.so (CUDA kernels + C-ABI) in-tree with nvcc for sm_100a.

`python -m paper_2203_11100_b200.build` or `build_library()`.  The library lands next to this file
so that it travels with the repository snapshot; nothing is installed into site-packages.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libswb200.so"
SOURCES = ["cabi.cu", "pack.cpp"]
HEADERS = ["kernels.cuh", "pipeline.cuh", "duo.cuh", "duo.inl", "scan_plan.hpp", "pipe_rates.cuh", "pack.hpp", "plan.inl", "handle.inl", "scan.inl", "persist.inl", "pairs.inl", "pipe.inl",
           "multi.inl"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo",
    "-Xcompiler", "-fPIC,-O3,-Wall,-Wno-unused-function",
    "-shared", "-cudart", "static",
]


KERNEL_SOURCES = ["kernels.cuh", "pipeline.cuh", "duo.cuh"]


def kernel_source_hash() -> str:
    """sha256 over the device code of the scan kernels: ncu-derived numbers that bench.py quotes (profiles/traffic.json)
    are stamped with it and dropped when the kernels have changed since the capture."""
    import hashlib
    h = hashlib.sha256()
    for name in KERNEL_SOURCES:
        h.update((CSRC / name).read_bytes())
    return h.hexdigest()


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; libswb200.so must be prebuilt")


def is_stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / f for f in SOURCES + HEADERS] + [PKG.parent / "include" / "swb200.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and not is_stale():
        return LIB
    extra = [f"-D{k}={os.environ[k]}" for k in ("SWB_INTER_TILE", "SWB_INTER_THREADS", "SWB_PIPE_STATS", "SWB_PIPE_POLL_NS") if k in os.environ]   # tuning only
    out = Path(os.environ.get("SWB_LIB_OUT", str(LIB)))
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-ccbin", "/usr/bin/g++", "-o", str(out)] + [str(CSRC / s) for s in SOURCES] + ["-ldl", "-lpthread"]
    if verbose:
        cmd.insert(1, "-Xptxas")
        cmd.insert(2, "-v")
        print(" ".join(cmd))
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libswb200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    return LIB


if __name__ == "__main__":
    build_library(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
