"""Config 5: where the collide time goes — the colliding poses vs the rest,
each subset timed alone (median of 5) with its stats (BV tests, leaf pairs,
triangle tests).  Usage: python tools/work_split.py [config]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_05348_b200 as M
from workloads import generators as G

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
w = G.make_config(cfg)
A = M.build_compressed_bvh(w.A.vertices, w.A.triangles, w.branching, w.bits, w.treelet).to_device()
B = M.build_compressed_bvh(w.B.vertices, w.B.triangles, w.branching, w.bits, w.treelet).to_device()
P = torch.from_numpy(w.poses).cuda()
ws = M.Workspace(A, B, 0)
hit, cnt = M.collide_batch(A, B, P, workspace=ws)
M.check(ws)
c = cnt.cpu().numpy().view(np.uint32).astype(np.int64)


def run(idx, reps=5):
    Q = P[torch.from_numpy(np.ascontiguousarray(idx)).cuda()].contiguous()
    M.collide_batch(A, B, Q, workspace=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        M.collide_batch(A, B, Q, workspace=ws)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    M.collide_batch(A, B, Q, workspace=ws, stats=True)
    st = M.read_stats(ws)
    st.pop("timeline_ns", None)
    return {"n": int(len(idx)), "ms": float(np.median(ts)), **{k: st[k] for k in ("bv_tests", "leaf_pairs", "tri_tests", "expansions")}}


out = {"config": cfg, "pairs_total": int(c.sum())}
out["all"] = run(np.arange(len(c)))
out["colliding"] = run(np.nonzero(c > 0)[0])
out["noncolliding"] = run(np.nonzero(c == 0)[0])
print(json.dumps(out))
