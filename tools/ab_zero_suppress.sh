#!/bin/bash
# f4: zero-suppressed (integer-compressed) corrections vs the plain layouts (ms / step, hierarchy bytes)
for cfg in ${CONFIGS:-5 3 2}; do
  for v in "" "--align-treelets --staging off" "--zero-suppress --staging off" "--zero-suppress --staging on"; do
    timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --quick $v 2>&1 | tail -1 | python -c "
import sys, json
l = sys.stdin.read().strip()
try:
    d = json.loads(l); print('cfg$cfg', '${v:-packed}'.ljust(32), round(d['ms_per_step'], 3), 'ms', 'B/node', {k: round(x, 2) for k, x in d['bytes_per_node'].items()}, 'bvh_bytes', d.get('bvh_bytes'), 'blocks', d.get('treelet_blocks'))
except Exception:
    print('cfg$cfg', '$v', 'FAILED', l[-300:])
"
  done
done
