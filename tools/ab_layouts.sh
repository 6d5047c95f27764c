#!/bin/bash
# the paper's §IV comparison on B200: delta vs binary16 vs fp32 node boxes
for cfg in ${CONFIGS:-5 2 3}; do
  for lay in delta fp16 fp32; do
    timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --quick --layout $lay 2>&1 | tail -1 | python -c "
import sys, json
l = sys.stdin.read().strip()
try:
    d = json.loads(l); print('cfg$cfg', '$lay', round(d['ms_per_step'], 3), 'ms', round(d['value'] / 1e6, 3), 'M/s', 'bv_tests', d['bv_tests'], 'B/node', {k: round(v, 2) for k, v in d['bytes_per_node'].items()})
except Exception:
    print('cfg$cfg', '$lay', 'FAILED', l[-300:])
"
  done
done
