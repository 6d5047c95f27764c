#!/bin/bash
# phase schedules on the full configs: tools/ab_phases_full.sh "32,32,64" "32,64" ...
for cfg in ${CONFIGS:-5 3 2}; do
  for s in "$@"; do
    CBVH_PHASES=$s python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --quick 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('cfg$cfg CBVH_PHASES=$s', round(d['ms_per_step'], 3), 'ms launches', d['launches'], 'dumped', d['dumped'])"
  done
done
