#!/bin/bash
# BASELINE config 3: branching x correction width sweep (poses/s, bytes/node)
for B in 2 4 8; do
  for b in 4 8 16; do
    timeout 600 python bench.py --config 3 --branching $B --bits $b --steps 3 --warmup 3 --quick 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print(json.dumps({'B': $B, 'bits': $b, 'ms_per_step': round(d['ms_per_step'], 3), 'poses_per_s': round(d['value']), 'bv_tests': d['bv_tests'], 'bytes_per_node': {k: round(v, 2) for k, v in d['bytes_per_node'].items()}}))"
  done
done
