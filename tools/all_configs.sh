#!/bin/bash
# Per-config timing of the default library (DESIGN.md §5 results table).
run() {
  timeout 600 python bench.py "$@" --steps 5 --warmup 3 --quick 2>&1 | tail -1 | python -c "
import sys, json
l = sys.stdin.read().strip()
try:
    d = json.loads(l); print('$*'.ljust(44), round(d['ms_per_step'], 3), 'ms', round(d['value'] / 1e6, 4), 'M poses/s', 'bv', d.get('bv_tests'), 'leaf', d.get('leaf_pairs'), 'tri', d.get('tri_tests'), 'exact', d.get('exact_tests'))
except Exception:
    print('$*', 'FAILED', l[-300:])
"
}
run --config 1
run --config 2
run --config 3
run --config 4
run --config 5
run --config 5 --early-exit
run --config 1 --preset contact
run --config 1 --preset contact --mode distance
run --config 3 --preset contact
run --config 3 --preset contact --mode distance
