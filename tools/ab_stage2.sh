#!/bin/bash
# staging variants: library (slots) x sides, aligned blobs
for cfg in ${CONFIGS:-5 3}; do
  for lib in libcbvh_cur.so libcbvh_st8.so libcbvh_st2.so; do
    for sides in 3 1 2; do
      CBVH_STAGE_SIDES=$sides CBVH_LIB=$PWD/paper_2012_05348_b200/$lib timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --quick --align-treelets --staging on 2>&1 | tail -1 | python -c "
import sys, json
l = sys.stdin.read().strip()
try:
    d = json.loads(l); print('cfg$cfg', '$lib', 'sides $sides', round(d['ms_per_step'], 3), 'ms', 'blocks', d.get('treelet_blocks'), 'staged', d.get('staged_reads'), 'decoded', d.get('nodes_decoded'))
except Exception:
    print('cfg$cfg', '$lib', 'FAILED', l[-300:])
"
    done
  done
done
