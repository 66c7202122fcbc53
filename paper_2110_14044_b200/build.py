"""Build libials_b200.so in-tree with nvcc for sm_100a (no torch extension
machinery; the library is a plain C ABI loaded with ctypes)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libials_b200.so")
# bounds-checked variant (-DIALS_CHECKS: device asserts on every index-driven
# gather / scatter of the sweeps); loaded instead when IALS_LIB=checked
OUT_CHECKED = os.path.join(HERE, "libials_b200_checked.so")
SOURCES = ["ials_abi.cu"]
DEPS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh")))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-I", os.path.join(ROOT, "include"),
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def up_to_date(out=OUT) -> bool:
    if not os.path.exists(out):
        return False
    t = os.path.getmtime(out)
    files = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(ROOT, "include", "ials_b200.h")]
    return all(os.path.getmtime(f) <= t for f in files)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    out = OUT_CHECKED if checked else OUT
    if not force and up_to_date(out):
        return out
    cmd = [nvcc(), *NVCC_FLAGS, *(["-DIALS_CHECKS"] if checked else []), "-o", out + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES], "-ldl"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
