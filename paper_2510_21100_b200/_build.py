"""Build the in-tree C-ABI shared library libhistretinex.so (nvcc, sm_100a)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = ["csrc/hr_api.cu", "csrc/k_hist.cu", "csrc/k_solve.cu", "csrc/k_apply.cu", "csrc/k_quality.cu"]
HEADERS = ["../include/histretinex.h"]  # + every csrc/*.cuh (see stale())
LIB = os.path.join(HERE, "libhistretinex.so")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "--cudart", "static",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def stale() -> bool:
    """True when the library is missing or older than any source or header it is built from."""
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = SOURCES + HEADERS + [os.path.join("csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))
                                if f.endswith((".cuh", ".h"))]
    return any(os.path.getmtime(os.path.join(HERE, f)) > t for f in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", tmp, *[os.path.join(HERE, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd, cwd=HERE)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
