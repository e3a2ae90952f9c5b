"""Build libsmc.so (the C-ABI library) in-tree for sm_100a with nvcc.

Run as a script (``python paper_2112_00364_b200/csrc/build.py``) or load by
path; it does not import the package (whose import needs the library)."""
from __future__ import annotations

import glob
import os
import subprocess

CSRC = os.path.dirname(os.path.abspath(__file__))
HERE = os.path.dirname(CSRC)
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libsmc.so")
SRC = os.path.join(CSRC, "engine.cu")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*")) +
                  [os.path.join(ROOT, "include", "smc.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    if not os.path.exists(nvcc) and os.path.exists("/usr/local/cuda/bin/nvcc"):
        nvcc = "/usr/local/cuda/bin/nvcc"
    cmd = [nvcc, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           "-o", LIB + ".tmp", SRC]
    extra = os.environ.get("SMC_NVCC_FLAGS", "").split()
    cmd[1:1] = extra
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
