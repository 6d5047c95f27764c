#!/bin/bash
# k-DOP bounding volumes on the static model B (Table I): 6 (AABB) / 14 / 18 / 26
for cfg in ${CONFIGS:-5 2 3 1}; do
  for k in 6 14 18 26; do
    timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --quick --kdop $k $EXTRA 2>&1 | tail -1 | python -c "
import sys, json
l = sys.stdin.read().strip()
try:
    d = json.loads(l); print('cfg$cfg', 'k=$k', round(d['ms_per_step'], 3), 'ms', round(d['value'] / 1e6, 3), 'M/s', 'bv', d['bv_tests'], 'leaf', d['leaf_pairs'], 'tri', d['tri_tests'], 'B/node', {k: round(v, 2) for k, v in d['bytes_per_node'].items()})
except Exception:
    print('cfg$cfg', 'k=$k', 'FAILED', l[-300:])
"
  done
done
