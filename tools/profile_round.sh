#!/bin/bash
# Run on the GPU box (via gpurun): launch list of the bench command, and one
# full ncu capture of the dominant kernel (phase 0 of traverse_kernel).
set -x
OUT=gpurun_out
CMD_LIST="python bench.py --steps 5 --warmup 3 --no-cpu"
CMD_FULL="python bench.py --steps 1 --warmup 3 --no-cpu --quick"
$CMD_LIST > $OUT/plain_list.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD_LIST > $OUT/ncu_list.log 2>&1
$CMD_FULL > $OUT/plain_full.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:traverse -s 4 -c 1 -o $OUT/prof $CMD_FULL > $OUT/ncu_full.log 2>&1
echo done
