#!/bin/bash
OUT=gpurun_out
CMD="python bench.py --config 4 --poses 8192 --steps 1 --warmup 3 --no-cpu --quick"
$CMD > $OUT/plain_dist.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:traverse -s 4 -c 1 -o $OUT/prof_dist $CMD > $OUT/ncu_dist.log 2>&1
echo done
