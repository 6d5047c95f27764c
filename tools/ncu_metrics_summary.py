"""Summarise `ncu --metrics ... --csv` launch lists of configs 1-3 (the four
phases of one collide call) into profiles/roundN_ncu_configs1-3.json.

usage: python tools/ncu_metrics_summary.py out.json cfg1=metrics1.csv cfg2=... """
import csv
import json
import sys
from collections import defaultdict


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    per = defaultdict(dict)
    for r in rows:
        per[int(r[0])][r[12]] = float(r[14].replace(",", ""))
    return [per[k] for k in sorted(per)]


def main(out, specs):
    d = {}
    for s in specs:
        key, path = s.split("=")
        L = load(path)
        p0 = L[0]
        d[key] = {"phase0": {
            "kernel_ms": p0["gpu__time_duration.sum"] / 1e6,
            "lts_GBps": p0["lts__t_bytes.sum.per_second"] / 1e9 if p0["lts__t_bytes.sum.per_second"] > 1e6 else p0["lts__t_bytes.sum.per_second"],
            "lts_bytes": p0["lts__t_bytes.sum"],
            "dram_GBps": p0["dram__bytes.sum.per_second"] / 1e9 if p0["dram__bytes.sum.per_second"] > 1e6 else p0["dram__bytes.sum.per_second"],
            "dram_bytes": p0["dram__bytes.sum"],
            "warp_exec_efficiency": p0["smsp__thread_inst_executed_per_inst_executed.ratio"] / 32,
            "issue_active_pct": p0["smsp__issue_active.avg.pct_of_peak_sustained_active"],
            "warps_active_pct": p0["sm__warps_active.avg.pct_of_peak_sustained_active"],
            "sm_active_over_elapsed": p0["sm__cycles_active.avg"] / p0["sm__cycles_elapsed.avg"]},
            "phases_captured": len(L), "phase_ms": [x["gpu__time_duration.sum"] / 1e6 for x in L]}
    d["source"] = ("tools/profile_final.sh: ncu --metrics ... --clock-control none -k regex:traverse -s 4 -c 4 on "
                   "`bench.py --quick --config k` (the phases of the second collide call)")
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
