#!/bin/bash
# Phase schedules (CBVH_PHASES, budgets of the bounded phases) on small batches
# and on configs 2 / 5: tools/ab_phases_small.sh "32,32,64" "4,4,8,16,32,64" ...
for s in "$@"; do
  echo "== CBVH_PHASES=$s"
  for c in 1 3 4; do CBVH_PHASES=$s python tools/small_batch.py $c 64 1024 16384 2>&1 | grep -v "^$"; done
  for c in 2 5; do CBVH_PHASES=$s python bench.py --config $c --steps 5 --warmup 3 --quick 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('cfg$c full', round(d['ms_per_step'], 3), 'ms launches', d['launches'])"; done
done
