#!/bin/bash
# Run on the GPU box (via gpurun): bench, launch list, one full ncu capture.
set -x
OUT=gpurun_out
CMD_LIST="python bench.py --steps 5 --warmup 3 --no-cpu"
CMD_FULL="python bench.py --steps 1 --warmup 3 --no-cpu --poses 262144"
$CMD_LIST > $OUT/plain_list.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD_LIST > $OUT/ncu_list.log 2>&1
$CMD_FULL > $OUT/plain_full.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:traverse -s 3 -c 1 -o $OUT/prof $CMD_FULL > $OUT/ncu_full.log 2>&1
echo done
