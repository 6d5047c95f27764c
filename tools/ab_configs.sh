#!/bin/bash
# quick timing of every config under phase schedules: tools/ab_configs.sh "sched1" "sched2"
for sched in "$@"; do
  for cfg in 1 2 3 4 5; do
    CBVH_PHASES="$sched" timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --quick 2>&1 | tail -1 | sed "s/^/[cfg$cfg $sched] /" | cut -c1-200
  done
done
