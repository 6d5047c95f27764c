"""Distance headroom: config-4 distance_batch from +inf vs capped just above
the answer (an ideal start) — time and BV tests.  Usage: python tools/dist_caps.py [config] [poses]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_05348_b200 as M
from workloads import generators as G

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = G.make_config(cfg, num_poses=n)
A = M.build_compressed_bvh(w.A.vertices, w.A.triangles, w.branching, w.bits, w.treelet).to_device()
B = M.build_compressed_bvh(w.B.vertices, w.B.triangles, w.branching, w.bits, w.treelet).to_device()
P = torch.from_numpy(w.poses).cuda()
ws = M.Workspace(A, B, 1)


def run(caps=None, reps=3):
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        d = M.distance_batch(A, B, P, workspace=ws, caps=caps)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    M.check(ws)
    M.distance_batch(A, B, P, workspace=ws, caps=caps, stats=True)
    st = M.read_stats(ws)
    return d.clone(), {"ms": float(np.median(ts[1:])), **{k: st[k] for k in ("bv_tests", "leaf_pairs", "tri_tests", "exact_tests", "iterations")}}


d0, r0 = run()
caps = d0 * (1 + 2e-5) + 1e-6
d1, r1 = run(caps)
print(json.dumps({"config": cfg, "free": r0, "ideal_cap": r1,
                  "max_rel_diff": float(((d1 - d0).abs() / d0.clamp_min(1e-6)).max())}))
