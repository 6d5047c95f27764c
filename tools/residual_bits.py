"""How compressible are the b-bit corrections?  Histogram of the stored
corrections' bit lengths and the bytes per node a per-sibling-group
bit-packing (frame-of-reference width per group + 4-bit width tag) would
need — the "integer compression" of P:204."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_05348_b200 as M  # noqa: E402
from workloads import generators as G  # noqa: E402

for cfg in (5, 3, 2):
    w = G.make_config(cfg, num_poses=1)
    for name, mesh in (("A", w.A), ("B", w.B)):
        bv = M.build_compressed_bvh(mesh.vertices, mesh.triangles, w.branching, w.bits, w.treelet)
        i = bv.info
        n = i["num_nodes"]
        codes = bv.blob[i["off_codes"]:i["off_codes"] + 6 * n].reshape(n, 6).astype(np.int64)
        topo = np.frombuffer(bv.blob[i["off_topo"]:i["off_topo"] + 4 * n].tobytes(), np.uint32)
        bl = np.zeros_like(codes)
        nz = codes > 0
        bl[nz] = np.floor(np.log2(codes[nz])).astype(np.int64) + 1
        bits = 0
        for p in np.nonzero((topo >> 31) == 0)[0]:
            f, c = int(topo[p] & 0x0FFFFFFF), int(((topo[p] >> 28) & 7) + 1)
            bits += 6 * c * int(bl[f:f + c].max()) + 4
        print(f"config {cfg} {name}: {n} nodes, mean correction bit length {bl.mean():.2f}, "
              f"fraction by bit length {np.round(np.bincount(bl.ravel(), minlength=9)[:9] / bl.size, 3).tolist()}, "
              f"group-packed {bits / 8 / n:.2f} B/node vs {6 * w.bits / 8:.0f} B fixed")
