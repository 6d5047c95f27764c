#!/bin/bash
# A/B of library variants on distance workloads: tools/ab_dist.sh lib1.so lib2.so ...
for args in "--config 4" "--config 3 --mode distance --poses 32768" "--config 3 --preset contact --mode distance --poses 16384" "--config 2 --mode distance --poses 16384"; do
  for v in "$@"; do
    CBVH_LIB=$PWD/paper_2012_05348_b200/$v timeout 600 python bench.py $args --steps 3 --warmup 3 --quick 2>&1 | tail -1 | python -c "
import sys, json
l = sys.stdin.read().strip()
try:
    d = json.loads(l); print('$args'.ljust(52), '$v', round(d['ms_per_step'], 3), 'ms', 'bv', d.get('bv_tests'), 'leaf', d.get('leaf_pairs'), 'tri', d.get('tri_tests'), 'exact', d.get('exact_tests'))
except Exception:
    print('$args', '$v', 'FAILED', l[-300:])
"
  done
done
