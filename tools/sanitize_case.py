"""Small collide + distance runs for compute-sanitizer (configs 1 and 3, few poses)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2012_05348_b200 as M
from workloads import generators as G

for k, n in ((1, 256), (3, 64)):
    w = G.make_config(k, num_poses=n)
    A = M.build_compressed_bvh(w.A.vertices, w.A.triangles, w.branching, w.bits, w.treelet).to_device()
    B = M.build_compressed_bvh(w.B.vertices, w.B.triangles, w.branching, w.bits, w.treelet).to_device()
    P = torch.from_numpy(w.poses).cuda()
    ws = M.Workspace(A, B, 0)
    h, c = M.collide_batch(A, B, P, workspace=ws)
    M.check(ws)
    h2, c2 = M.collide_batch(A, B, P, workspace=ws, early_exit=True, stats=True)
    M.check(ws)
    wd = M.Workspace(A, B, 1)
    d = M.distance_batch(A, B, P[:32], workspace=wd)
    M.check(wd)
    print(k, int(h.sum()), int(c.sum()), float(d.min()))
print("sanitize case ok")
