"""Build libdog.so (the sm_100a CUDA library behind include/dog.h) in-tree with nvcc."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.environ.get("DOG_CSRC") or os.path.join(PKG, "csrc")   # DOG_CSRC: alternative sources (A/B)
LIB = os.environ.get("DOG_LIB") or os.path.join(PKG, "libdog.so")
SOURCES = ["dog.cu"]
HEADERS = ["dog_common.cuh", "dog_rng.cuh", "dog_kernels.cuh", "dog_cells.cuh", "dog_resample.cuh", "dog_sort.cuh", "dog_fcount.cuh", "dog_ego.cuh", "dog_eval.cuh", "dog_doppler.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    # no --use_fast_math: the parity path relies on IEEE division/sqrt and explicit _rn intrinsics
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "dog.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = LIB + f".tmp{os.getpid()}"
    extra = os.environ.get("DOG_NVCC_EXTRA", "").split()   # diagnostics builds only (e.g. -DDOG_TIMING)
    cmd = [nvcc, *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
