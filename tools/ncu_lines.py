"""Aggregate an ncu `--page source --print-source=cuda,sass` CSV by CUDA source line.

usage: ncu -i prof.ncu-rep --page source --csv --print-source=cuda,sass > x.csv
       python tools/ncu_lines.py x.csv [top]
"""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    agg = defaultdict(lambda: [0, 0, 0, ""])
    cur_file, cur_line, cur_src = "", None, ""
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            cur_line, cur_src = r[0], r[1]
        try:
            samples = int(r[4] or 0)
            inst = int(r[7] or 0)
            thr = int(r[8] or 0)
        except ValueError:
            continue
        a = agg[(cur_file, cur_line)]
        a[0] += samples
        a[1] += inst
        a[2] += thr
        a[3] = cur_src.strip()[:80]
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_i = sum(v[1] for v in agg.values()) or 1
    print(f"total stall samples {tot_s}, warp instructions {tot_i}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        eff = v[2] / (32 * v[1]) if v[1] else 0
        print(f"{k[0]:>18}:{k[1]:<5} samp {100*v[0]/tot_s:5.1f}%  inst {100*v[1]/tot_i:5.1f}%  simt {eff:4.2f}  {v[3]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
