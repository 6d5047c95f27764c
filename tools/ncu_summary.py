"""Summarise one kernel of an `ncu --page raw --csv` export into the JSON kept
under profiles/ (throughputs, IPC, occupancy, SIMT efficiency, cache hit
rates, DRAM bytes, L2->L1 traffic, stall reasons per issue).

usage: ncu -i prof.ncu-rep --page raw --csv > raw.csv
       python tools/ncu_summary.py raw.csv [row] > profiles/roundN_....json
"""
import csv
import json
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes.sum.per_second",
    "lts__t_sectors.sum",
    "lts__t_sectors.sum.per_second",
]


def main(path, row=0):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2 + row]
    col = {h: i for i, h in enumerate(hdr)}
    out = {"kernel": vals[col["Kernel Name"]]}
    for k in KEYS:
        if k in col:
            out[k] = f"{vals[col[k]]} {units[col[k]]}".strip()
    stalls = {}
    for h, i in col.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                v = float(vals[i])
            except ValueError:
                continue
            if v >= 0.05:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
    out["stall_reasons_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
