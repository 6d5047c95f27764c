#!/bin/bash
# The paper's half- vs single-precision comparison on its own
# preset: the zero-separation poses found by bisection (configs 1 and 3),
# collide and distance, delta / fp16 / fp32 node boxes (ms / step).
for cfg in 1 3; do
  for mode in collide distance; do
    for layout in delta fp16 fp32; do
      timeout 600 python bench.py --config $cfg --preset zero --mode $mode --layout $layout --steps 5 --warmup 3 --quick 2>&1 | tail -1 | python -c "
import sys, json
l = sys.stdin.read().strip()
try:
    d = json.loads(l); print('cfg$cfg zero $mode $layout'.ljust(34), round(d['ms_per_step'], 3), 'ms', round(d['value'] / 1e6, 4), 'M poses/s', 'bv', d.get('bv_tests'), 'B/node', d.get('bytes_per_node'))
except Exception:
    print('cfg$cfg $mode $layout', 'FAILED', l[-300:])
"
    done
  done
done
