"""Build libraduls_gpu.so in-tree with nvcc for sm_100a.

    python -m paper_1612_02557_b200.build [--verbose]

The library is a plain C-ABI shared object (include/raduls_gpu.h): no torch
types, no Python extension module. It is git-ignored and travels to the GPU
box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libraduls_gpu.so")
SOURCES = [os.path.join(CSRC, "raduls_gpu.cu")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _deps() -> list[str]:
    out = list(SOURCES)
    for f in os.listdir(CSRC):
        if f.endswith((".cuh", ".h")):
            out.append(os.path.join(CSRC, f))
    out.append(os.path.join(ROOT, "include", "raduls_gpu.h"))
    return out


LIB_CHECKED = os.path.join(HERE, "libraduls_gpu_checked.so")


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in _deps())


def build(verbose: bool = False, force: bool = False, checked: bool = False) -> str:
    """libraduls_gpu.so, or (checked=True) libraduls_gpu_checked.so: the same
    sources with -DRG_CHECKED (bounds/alignment checks on every global record
    access, bounded mbarrier waits, poisoned scratch and shared memory,
    optional scheduling jitter; see csrc/common.cuh) — the race/bounds
    evidence on a pool without compute-sanitizer."""
    lib = LIB_CHECKED if checked else LIB
    if not force and not needs_build(lib):
        return lib
    cmd = [NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
           "-shared", "-cudart", "static", "-I", os.path.join(ROOT, "include"),
           *(["-DRG_CHECKED"] if checked else []),
           "-o", lib + ".tmp", *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    os.replace(lib + ".tmp", lib)
    if verbose:
        sys.stderr.write(res.stderr)
    return lib


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force=True, checked="--checked" in sys.argv))
