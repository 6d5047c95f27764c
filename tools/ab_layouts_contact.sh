#!/bin/bash
# the paper's §IV experiment setting: the zero-distance preset, half vs
# float node boxes — collide and distance, configs 3 and 1
for cfg in ${CONFIGS:-3 1}; do
  for mode in collide distance; do
    for lay in delta fp16 fp32; do
      timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --quick --preset contact --mode $mode --layout $lay 2>&1 | tail -1 | python -c "
import sys, json
l = sys.stdin.read().strip()
try:
    d = json.loads(l); print('cfg$cfg', 'contact', '$mode', '$lay', round(d['ms_per_step'], 3), 'ms', round(d['value'] / 1e6, 4), 'M/s', 'bv', d['bv_tests'], 'B/node', {k: round(v, 2) for k, v in d['bytes_per_node'].items()})
except Exception:
    print('cfg$cfg', '$mode', '$lay', 'FAILED', l[-300:])
"
    done
  done
done
