#!/bin/bash
# A/B of phase schedules: tools/ab_phases.sh "32,32,64" "-1" ...
for v in "$@"; do
  CBVH_PHASES="$v" timeout 300 python bench.py --steps 10 --warmup 3 --quick 2>&1 | tail -1 | sed "s/^/[$v] /"
done
