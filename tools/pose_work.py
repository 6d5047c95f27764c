"""Per-pose work distribution on config 5: pair-count percentiles and the
device time of the heaviest / median colliding poses run alone."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_05348_b200 as M
from workloads import generators as G

w = G.make_config(5)
A = M.build_compressed_bvh(w.A.vertices, w.A.triangles, 4, 8, 64).to_device()
B = M.build_compressed_bvh(w.B.vertices, w.B.triangles, 4, 8, 64).to_device()
P = torch.from_numpy(w.poses).cuda()
ws = M.Workspace(A, B, 0)
hit, cnt = M.collide_batch(A, B, P, workspace=ws)
M.check(ws)
c = cnt.cpu().numpy().astype(np.int64)
col = c[c > 0]
out = {"colliding": int(len(col)), "pct": {q: int(np.percentile(col, q)) for q in (50, 90, 99, 99.9, 100)}}
order = np.argsort(-c)


def time_subset(idx, reps=3):
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
    return min(ts)


out["top1_ms"] = time_subset(order[:1])
out["top10_ms"] = time_subset(order[:10])
out["top100_ms"] = time_subset(order[:100])
med = np.nonzero(c > 0)[0]
med = med[np.argsort(c[med])][len(med) // 2: len(med) // 2 + 100]
out["median100_ms"] = time_subset(med)
out["noncolliding100_ms"] = time_subset(np.nonzero(c == 0)[0][:100])
st = {}
for k, idx in (("top1", order[:1]), ("median1", med[:1])):
    Q = P[torch.from_numpy(np.ascontiguousarray(idx)).cuda()].contiguous()
    M.collide_batch(A, B, Q, workspace=ws, stats=True)
    st[k] = M.read_stats(ws)
    st[k].pop("timeline_ns")
out["stats"] = st
print(json.dumps(out))
