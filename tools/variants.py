#!/usr/bin/env python
"""Build A/B variants of libcbvh.so side by side (tuning only, not the product).

    python tools/variants.py name:-DFLAG=1,-DOTHER=2 name2: ...
    python tools/variants.py --rev r1=6bcbcb6      # the library as of a git revision

Each variant is paper_2012_05348_b200/libcbvh_<name>.so, compiled with the
product's nvcc flags plus the given -D flags; run them with tools/ab.sh.
"""
import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2012_05348_b200 import build as B  # noqa: E402


def compile_variant(name, flags, csrc=B.CSRC):
    out = os.path.join(ROOT, "paper_2012_05348_b200", f"libcbvh_{name}.so")
    cmd = ["nvcc", *B.NVCC_FLAGS, *flags, "-o", out] + [os.path.join(csrc, s) for s in B.SOURCES]
    subprocess.check_call(cmd, cwd=csrc)
    return out


def compile_rev(name, rev):
    d = tempfile.mkdtemp()
    subprocess.check_call(f"git -C {ROOT} archive {rev} paper_2012_05348_b200/csrc include | tar -x -C {d}", shell=True)
    return compile_variant(name, [], os.path.join(d, "paper_2012_05348_b200", "csrc"))


def main(argv):
    jobs = []
    with ThreadPoolExecutor(8) as ex:
        it = iter(argv)
        for a in it:
            if a == "--rev":
                name, rev = next(it).split("=")
                jobs.append(ex.submit(compile_rev, name, rev))
            else:
                name, _, fl = a.partition(":")
                jobs.append(ex.submit(compile_variant, name, [f for f in fl.split(",") if f]))
        for j in jobs:
            print(j.result())


if __name__ == "__main__":
    main(sys.argv[1:])
