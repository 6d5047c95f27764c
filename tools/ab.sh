#!/bin/bash
# A/B timing of library variants on the same box: CONFIGS="5 3" tools/ab.sh lib1.so lib2.so ...
CONFIGS=${CONFIGS:-5}
for cfg in $CONFIGS; do
  for v in "$@"; do
    CBVH_LIB=$PWD/paper_2012_05348_b200/$v timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --quick $EXTRA 2>&1 | tail -1 | python -c "
import sys, json
l = sys.stdin.read().strip()
try:
    d = json.loads(l); print('cfg$cfg', '$v', round(d['ms_per_step'], 3), 'ms', round(d['value'] / 1e6, 3), 'M/s', 'lane_util', round(d.get('lane_util', 0), 3), 'iters', d.get('iterations'), 'bv', d.get('bv_tests'), 'leaf', d.get('leaf_pairs'), 'tri', d.get('tri_tests'), 'exact', d.get('exact_tests'))
except Exception:
    print('cfg$cfg', '$v', 'FAILED', l[-300:])
"
  done
done
