"""Aggregate ncu source-view samples into code regions given line ranges.
usage: python tools/ncu_regions.py cs.csv 'name:lo-hi,...'"""
import csv
import sys
from collections import defaultdict


def main(path, spec):
    ranges = []
    for item in spec.split(","):
        name, rng = item.split(":")
        lo, hi = rng.split("-")
        ranges.append((name, int(lo), int(hi)))
    rows = list(csv.reader(open(path)))
    agg = defaultdict(lambda: [0, 0])
    cur, hdr, f = ("", 0), None, ""
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            cur = (f, int(r[0]))
        try:
            s, i = int(r[4] or 0), int(r[7] or 0)
        except ValueError:
            continue
        fn, l = cur
        reg = "other:" + fn
        if fn == "cbvh_device.cu":
            for name, lo, hi in ranges:
                if lo <= l <= hi:
                    reg = name
                    break
        elif fn == "leaf_geometry.cuh":
            reg = "leaf_geometry"
        agg[reg][0] += s
        agg[reg][1] += i
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:28s} samples {100 * v[0] / ts:5.1f}%  inst {100 * v[1] / ti:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
