"""Per-call totals of the production traversal kernel from an ncu launch list
(`--metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum`),
written into profiles/ncu_traffic.json next to the DRAM bytes of the full capture.

usage: python tools/launch_totals.py launches.csv cfg5 [phases_per_call=4] [source-name]"""
import csv
import json
import os
import sys
from collections import defaultdict

path, key = sys.argv[1], sys.argv[2]
phases = int(sys.argv[3]) if len(sys.argv) > 3 else 4
src = sys.argv[4] if len(sys.argv) > 4 else path
rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
per = defaultdict(lambda: defaultdict(float))
for r in rows:
    kid, name, metric, val = r[0], r[4], r[12], r[14]
    if any(t in name for t in ("traverse_kernel<0, 0, 0>", "traverse_kernel<0, false, 0>",
                               "traverse_kernel<0, false, 0, false>", "traverse_kernel<0, 0, 0, 0>")):
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
d.setdefault(key, {}).update(out)
d[key]["inst_source"] = (f"ncu launch list ({src}): smsp__inst_executed.sum and "
                         "smsp__thread_inst_executed.sum summed over the phases of each production collide call")
json.dump(d, open(p, "w"), indent=1)
