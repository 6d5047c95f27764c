#!/bin/bash
for v in "$@"; do
  CBVH_LIB=$PWD/paper_2012_05348_b200/$v timeout 600 python bench.py --config 4 --poses 16384 --steps 3 --warmup 3 --quick 2>&1 | tail -1 | cut -c1-100 | sed "s/^/cfg4 $v /"
done
