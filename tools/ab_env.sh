#!/bin/bash
# A/B of an environment switch on the same box: tools/ab_env.sh VAR "v1 v2 v1" [bench args...]
VAR=$1; VALS=$2; shift 2
for cfg in ${CONFIGS:-5}; do
  for v in $VALS; do
    env $VAR=$v python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --quick "$@" 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('cfg$cfg $VAR=$v', round(d['ms_per_step'], 3), 'ms', 'kernel', round(d['kernel_ms'], 3))"
  done
done
