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
PROBE_SOURCES = ["probe_l2.cu"]
OUT_PROBE = os.path.join(HERE, "libcbvh_probe.so")  # measurement utility (L2 read peak), not the hot path

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


def build_probe(force: bool = False) -> str:
    """The L2 read-bandwidth probe bench.py reports its L2 roofline against."""
    src = [os.path.join(CSRC, s) for s in PROBE_SOURCES]
    if force or not os.path.exists(OUT_PROBE) or any(os.path.getmtime(f) > os.path.getmtime(OUT_PROBE) for f in src):
        nvcc = os.environ.get("NVCC", "nvcc")
        subprocess.check_call([nvcc, *NVCC_FLAGS, "-o", OUT_PROBE, *src], cwd=CSRC)
    return OUT_PROBE


if __name__ == "__main__":
    print(build(force=True, verbose=True))
    print(build(force=True, checked=True))
    print(build_probe(force=True))
