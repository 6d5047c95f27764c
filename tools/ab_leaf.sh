#!/bin/bash
# leaf sizes of A and B separately (ablation): tools/ab_leaf.sh "4 4" "4 2" ...
for cfg in ${CONFIGS:-5 3 2}; do
  for ab in "$@"; do
    read -r la lb <<< "$ab"
    python bench.py --config $cfg --steps 5 --warmup 3 --quick --leaf-a $la --leaf-b $lb 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('cfg$cfg leafA=$la leafB=$lb', round(d['ms_per_step'], 3), 'ms bv', d['bv_tests'], 'leaf', d['leaf_pairs'], 'tri', d['tri_tests'])"
  done
done
