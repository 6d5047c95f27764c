#!/usr/bin/env python
"""Latency of small batches (the launch- and dive-bound regime): median time of
collide_batch / distance_batch over N poses of a config's meshes.
    CBVH_LIB=... python tools/small_batch.py [config] [N ...]      (MODES=collide,distance selects the queries)"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2012_05348_b200 as M  # noqa: E402
from workloads import generators as G  # noqa: E402


def main(cfg, sizes):
    w = G.make_config(cfg, num_poses=max(sizes))
    dev = torch.device("cuda", 0)
    A = M.build_compressed_bvh(w.A.vertices, w.A.triangles, w.branching, w.bits, w.treelet).to_device(dev)
    B = M.build_compressed_bvh(w.B.vertices, w.B.triangles, w.branching, w.bits, w.treelet).to_device(dev)
    P = torch.from_numpy(w.poses).to(dev)
    st = torch.cuda.current_stream(dev)
    for mode in os.environ.get("MODES", "collide,distance").split(","):
        ws = M.Workspace(A, B, 1 if mode == "distance" else 0, dev)
        for n in sizes:
            Pn = P[:n].contiguous()
            hit = torch.empty(n, dtype=torch.uint8, device=dev)
            cnt = torch.empty(n, dtype=torch.int32, device=dev)
            dst = torch.empty(n, dtype=torch.float32, device=dev)
            ts = []
            for it in range(25):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                if mode == "distance":
                    M.distance_batch(A, B, Pn, dst, ws)
                else:
                    M.collide_batch(A, B, Pn, hit, cnt, ws)
                b.record(st)
                b.synchronize()
                if it >= 5:
                    ts.append(a.elapsed_time(b) * 1e3)
            M.check(ws)
            print(f"cfg{cfg} {mode:8s} N={n:6d} median {statistics.median(ts):8.1f} us  min {min(ts):8.1f} us  "
                  f"launches {M.last_launch_count()}  lib {os.path.basename(os.environ.get('CBVH_LIB', 'default'))}", flush=True)


if __name__ == "__main__":
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    sizes = [int(x) for x in sys.argv[2:]] or [64, 1024, 16384]
    main(cfg, sizes)
