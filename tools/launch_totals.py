"""Per-call totals of the production traversal kernel from an ncu launch list
(`--metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum`),
written into profiles/ncu_traffic.json next to the DRAM bytes of the full capture.

usage: python tools/launch_totals.py launches.csv cfg5 [phases_per_call=4] [source-name]"""
import csv
import hashlib
import json
import os
import re
import sys
from collections import defaultdict

path, key = sys.argv[1], sys.argv[2]
phases = int(sys.argv[3]) if len(sys.argv) > 3 else 4
src = sys.argv[4] if len(sys.argv) > 4 else path
rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
per = defaultdict(lambda: defaultdict(float))
for r in rows:
    kid, name, metric, val = r[0], r[4], r[12], r[14]
    # the production collide instantiations: MODE 0, STATS off, AABB blobs (any STAGE / FAST)
    if re.search(r"traverse_kernel<\(?(int\))?0, \(?(bool\))?(0|false), \(?(int\))?0[,>]", name):
        per[kid][metric] = float(val.replace(",", ""))
n = len(per)
tot = defaultdict(float)
for m in per.values():
    for k, v in m.items():
        tot[k] += v
calls = n / phases
out = {"warp_inst_per_launch": tot["smsp__inst_executed.sum"] / calls,
       "thread_inst_per_warp_inst": tot["smsp__thread_inst_executed.sum"] / max(1.0, tot["smsp__inst_executed.sum"]),
       "kernel_ns_per_call_serialised": tot["gpu__time_duration.sum"] / calls,
       "launches": n}
print(json.dumps(out))
p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
d = json.load(open(p)) if os.path.exists(p) else {}
# the kernel sources these counts belong to: bench.py reports roofline_issue
# only while the committed counts match the sources it runs
csrc = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2012_05348_b200", "csrc")
h = hashlib.sha256()
for f in ("cbvh_device.cu", "leaf_geometry.cuh"):
    h.update(open(os.path.join(csrc, f), "rb").read())
out["kernel_source_sha256"] = h.hexdigest()
d.setdefault(key, {}).update(out)
d[key]["inst_source"] = (f"ncu launch list ({src}): smsp__inst_executed.sum and "
                         "smsp__thread_inst_executed.sum summed over the phases of each production collide call")
json.dump(d, open(p, "w"), indent=1)
