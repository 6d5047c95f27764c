#!/bin/bash
# Treelet staging A/B: packed blobs, aligned blobs unstaged, aligned blobs staged.
for cfg in ${CONFIGS:-5 3 2}; do
  for v in "" "--align-treelets --staging off" "--align-treelets --staging on"; do
    timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --quick $v $EXTRA 2>&1 | tail -1 | python -c "
import sys, json
l = sys.stdin.read().strip()
try:
    d = json.loads(l); print('cfg$cfg', '${v:-packed}'.ljust(34), round(d['ms_per_step'], 3), 'ms', 'blocks', d.get('treelet_blocks'), 'staged', d.get('staged_reads'), 'decoded', d.get('nodes_decoded'), 'lane_util', round(d.get('lane_util', 0), 3))
except Exception:
    print('cfg$cfg', '$v', 'FAILED', l[-300:])
"
  done
done
