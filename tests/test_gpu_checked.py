"""Memory-safety evidence without compute-sanitizer (closed on the GPU pool):
the checked build (-DCBVH_CHECKED) bounds-checks every node, triangle, pose
and queue index on the device and reports a violation as CBVH_EINTERNAL.

* the sanitizer case (configs 1 and 3, collide / early exit / stats /
  distance) runs clean under the checked build;
* a blob whose root points past the node array is caught on the device
  (host validation bypassed; the offending lane is dropped, so the run stays
  in bounds) — and by cbvh_bind's host validation otherwise
  (tests/test_builder.py::test_bind_rejects_corrupt_topology).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2012_05348_b200", "libcbvh_checked.so")


def _run(code_or_file, *args, timeout=300, extra_env=None):
    env = dict(os.environ, CBVH_LIB=CHECKED, **(extra_env or {}))
    cmd = [sys.executable] + ([code_or_file] if code_or_file.endswith(".py") else ["-c", code_or_file]) + list(args)
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_checked_build_runs_clean():
    assert os.path.exists(CHECKED), "build() must produce libcbvh_checked.so"
    r = _run(os.path.join(ROOT, "tools", "sanitize_case.py"))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "sanitize case ok" in r.stdout


CORRUPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2012_05348_b200 as M
from paper_2012_05348_b200 import _lib as L
from workloads import generators as G
w = G.make_config(1, num_poses=64)
A = M.build_compressed_bvh(w.A.vertices, w.A.triangles, 2, 8)
B = M.build_compressed_bvh(w.B.vertices, w.B.triangles, 2, 8).to_device()
off = A.info["off_topo"]
root = int(np.frombuffer(A.blob[off:off + 4].tobytes(), np.uint32)[0])
bad = (root & ~0x0FFFFFFF) | 0x0FFFFFF0        # first child far past the node array
A.blob[off:off + 4] = np.frombuffer(np.uint32(bad).tobytes(), np.uint8)
A.to_device()
ws = M.Workspace(A, B, 0)
M.collide_batch(A, B, torch.from_numpy(w.poses).cuda(), workspace=ws)
try:
    M.check(ws)
    print("NOT CAUGHT")
except L.CbvhError as e:
    print("CAUGHT", e.code)
"""


def test_checked_build_catches_bad_index():
    # host validation bypassed so the device-side checks see the bad index
    r = _run(CORRUPT, extra_env={"CBVH_SKIP_BLOB_VALIDATION": "1"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "CAUGHT -8" in r.stdout
