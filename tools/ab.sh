#!/bin/bash
# A/B timing of library variants on the same box: tools/ab.sh lib1.so lib2.so ...
for v in "$@"; do
  for rep in 1 2; do
    CBVH_LIB=$PWD/paper_2012_05348_b200/$v timeout 600 python bench.py --steps 10 --warmup 3 --quick "${AB_ARGS[@]}" 2>&1 | tail -1
  done
done
