"""Build libcbvh.so in-tree with nvcc for sm_100a (no JIT cache, no fallback)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["cbvh_device.cu", "builder.cpp"]
HEADERS = ["cbvh_internal.h", "leaf_geometry.cuh", os.path.join("..", "..", "include", "cbvh.h")]
OUT = os.path.join(HERE, "libcbvh.so")
OUT_CHECKED = os.path.join(HERE, "libcbvh_checked.so")  # -DCBVH_CHECKED: device bounds checks

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-shared"]


def _stale_at(out) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(os.path.join(CSRC, s)) > t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    out = OUT_CHECKED if checked else OUT
    if force or _stale_at(out):
        nvcc = os.environ.get("NVCC", "nvcc")
        cmd = [nvcc, *NVCC_FLAGS]
        if checked:
            cmd += ["-DCBVH_CHECKED"]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        cmd += ["-o", out] + [os.path.join(CSRC, s) for s in SOURCES]
        subprocess.check_call(cmd, cwd=CSRC)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
    print(build(force=True, checked=True))
