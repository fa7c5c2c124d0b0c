"""In-tree build of the sm_100a library (``_lib/libehmg_b200.so``).

nvcc cross-compiles here without a GPU; the built .so travels with the repo
snapshot to the B200 box.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.environ.get("EHMG_B200_LIB") or os.path.join(LIBDIR, "libehmg_b200.so")  # override: A/B builds
SOURCES = ["ehmg_solver.cu"]
HEADERS = ["ehmg_core.cuh", "ehmg_kernels.cuh", "ehmg_stencil2d.cuh", "ehmg_stencil3d.cuh", "ehmg_stencil3d_rr.cuh", "ehmg_stencil3d_sp.cuh", "ehmg_media.cuh", "ehmg_slab.cuh", "ehmg_comm.cuh", "ehmg_solver.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-diag-suppress", "177",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, h) for h in HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "ehmg_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if os.environ.get("EHMG_B200_LIB"):
        return LIB  # an A/B build chosen by the caller: never rebuilt here
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-o", LIB + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES],
           "-lcusolver", "-lcublas", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
