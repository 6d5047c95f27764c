#!/usr/bin/env python
"""Generate the zero-separation pose preset of configs 1 and 3 by bisection.

The paper's "most time consuming distance preset" is "a distance of zero"
between the two models (§IV); SPEC S:462 / S:487 build it by
bisection on the translation until |distance| < 1e-3.

For pose i the rotation and the unit translation direction u_i come from the
seeded draws of ``workloads.generators.zero_pose_draws`` (the config's pose
seed).  The translation magnitude s_i is bisected on [0, 2.2] with the fp64
oracle's distance (oracle/, nothing else): s_lo keeps distance 0 (the models
touch or overlap), s_hi keeps distance > 0, and the loop stops once
0 < distance(s_hi) < 1e-3.  Every distance is evaluated on the pose exactly
as the generator will produce it (fp64 R and s u, rounded to fp32 once), so
the stored s reproduce the oracle's values bit for bit.  Because a rigid
translation by ds moves every point by ds, distance is 1-Lipschitz in s, so
the bracket width bounds distance(s_hi) and 12 halvings always suffice.

Output: workloads/presets/zero_cfg{k}.npz with s (float64 [N]) and the
oracle distance at s (float64 [N]).

    python tools/make_zero_preset.py 1 1024
    python tools/make_zero_preset.py 3 32768
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from workloads import generators as G  # noqa: E402

TARGET = 1e-3
S_HI = 2.2  # radii <= 1.05 each: 2.2 apart the noisy unit spheres cannot touch


def main(k: int, n: int):
    w = G.make_config(k, num_poses=1)  # meshes only
    R, u = G.zero_pose_draws(k, n)
    tA = O.Tree.from_mesh(w.A.vertices, w.A.triangles)
    tB = O.Tree.from_mesh(w.B.vertices, w.B.triangles)

    def dist(idx, s):
        return O.distance(tA, tB, G.pack_poses(R[idx], s[:, None] * u[idx]))[0]

    lo = np.zeros(n)
    hi = np.full(n, S_HI)
    dhi = np.full(n, np.inf)
    t0 = time.time()
    idx = np.arange(n)
    d0 = dist(idx, lo)
    assert np.all(d0 == 0.0), f"{(d0 > 0).sum()} poses do not touch at s = 0"
    dhi = dist(idx, hi)
    assert np.all(dhi > 0), "poses touching at s = 2.2"
    for it in range(40):
        idx = np.nonzero(dhi >= TARGET)[0]
        if len(idx) == 0:
            break
        mid = 0.5 * (lo[idx] + hi[idx])
        dm = dist(idx, mid)
        z = dm == 0.0
        lo[idx[z]] = mid[z]
        hi[idx[~z]] = mid[~z]
        dhi[idx[~z]] = dm[~z]
        print(f"cfg{k} iter {it}: {len(idx)} poses open, {time.time() - t0:.0f} s", flush=True)
    assert np.all((dhi > 0) & (dhi < TARGET))
    out = os.path.join(ROOT, "workloads", "presets", f"zero_cfg{k}.npz")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    np.savez_compressed(out, s=hi, distance=dhi)
    print(out, "max distance", dhi.max(), "median", np.median(dhi), f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]))
