import numpy as np, torch, oracle as O, paper_2012_05348_b200 as M
from workloads import generators as G
Am, Bm, P = G.tiny_pair("8x4", seed=5, n_poses=3000, half_width=1.5)
tA, tB = O.Tree.from_mesh(Am.vertices, Am.triangles), O.Tree.from_mesh(Bm.vertices, Bm.triangles)
P = P[:500]
d64 = O.bruteforce_distance(tA, tB, P)
for Bf in (2,4,8):
    A = M.build_compressed_bvh(Am.vertices, Am.triangles, Bf, 8).to_device()
    B = M.build_compressed_bvh(Bm.vertices, Bm.triangles, Bf, 8).to_device()
    d = M.distance_batch(A, B, torch.from_numpy(P).cuda()).cpu().numpy().astype(np.float64)
    far = d64 > 1e-5
    rel = np.zeros_like(d64); rel[far] = np.abs(d[far]-d64[far])/d64[far]
    idx = np.argsort(-rel)[:6]
    print("B", Bf, [(int(i), float(d[i]), float(d64[i]), float(rel[i])) for i in idx])
