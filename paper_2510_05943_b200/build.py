"""Build libearl_dispatch.so in-tree for sm_100a (B200) with nvcc.

Usage: python -m paper_2510_05943_b200.build [--verbose]
The shared library is written next to this file; it is git-ignored but travels to the GPU box
with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libearl_dispatch.so")
SOURCES = ["api.cu", "planner.cu", "copy.cu", "aggregate.cu", "lengths.cu", "vmm.cu", "selector.cpp"]
HEADERS = ["earl_internal.cuh"]
PUBLIC_HEADER = os.path.join(ROOT, "include", "earl_dispatch.h")

def nccl_dir() -> str:
    """The NCCL torch ships with (same soname: one NCCL per process)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        d = list(spec.submodule_search_locations)[0]
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    return "/usr"


NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [PUBLIC_HEADER, __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nd = nccl_dir()
    cmd = [nvcc()] + NVCC_FLAGS + ["-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp"]
    if nd == "/usr":
        cmd += ["-lnccl"]
    else:
        cmd += ["-I", os.path.join(nd, "include"), "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
                "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
    # tuning experiments only (e.g. EARL_NVCC_DEFINES="EARL_AGG_CTAS_PER_SM=2")
    cmd += ["-D" + d for d in os.environ.get("EARL_NVCC_DEFINES", "").split()]
    cmd += [os.path.join(CSRC, s) for s in SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}): {' '.join(cmd)}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="--verbose" in sys.argv)
    print(LIB)
