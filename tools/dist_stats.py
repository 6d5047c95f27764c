import json, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2012_05348_b200 as M
import oracle as O
from workloads import generators as G
w = G.make_config(4, num_poses=int(sys.argv[1]) if len(sys.argv) > 1 else 2048)
A = M.build_compressed_bvh(w.A.vertices, w.A.triangles, 4, 8, 32).to_device()
B = M.build_compressed_bvh(w.B.vertices, w.B.triangles, 4, 8, 32).to_device()
P = torch.from_numpy(w.poses).cuda()
ws = M.Workspace(A, B, 1)
for descent in ("larger", "simultaneous"):
    d = M.distance_batch(A, B, P, workspace=ws, stats=True, descent=descent)
    M.check(ws)
    st = M.read_stats(ws); st.pop("timeline_ns")
    print(descent, json.dumps(st))
tA = O.Tree.from_mesh(w.A.vertices, w.A.triangles); tB = O.Tree.from_mesh(w.B.vertices, w.B.triangles)
t = time.time(); d64, ost = O.distance(tA, tB, w.poses[:64]); print("oracle 64 poses", time.time() - t, "s, bv_tests", ost)
