#!/bin/bash
# Round-2 final evidence (run on the GPU box via gpurun; one GPU, one process).
# Each profiled command first runs once without ncu and must exit 0; numbers
# printed under ncu are never bench values.
O=gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu"
Q="python bench.py --steps 1 --warmup 3 --no-cpu --quick"
# bench lines with the oracle leg and the in-run parity check, all five configs
python bench.py --csv $O/f_bench.csv > $O/f_bench_cfg5.json 2> $O/f_bench_cfg5.err
for k in 1 2 3 4; do python bench.py --config $k --steps 5 --warmup 3 --csv $O/f_bench.csv 2>> $O/f_bench_cfgs.err | tail -1 >> $O/f_bench_configs1-4.jsonl; done
# launch list of the bench command
$B > $O/f_plain.json 2> $O/f_plain.err && \
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum --clock-control none \
      --csv --log-file $O/f_launches_cfg5.csv $B > $O/f_ncu_list.log 2>&1
# full captures of the dominant kernel (phase 0 of the second call): collide config 5, distance config 4
$Q > $O/f_q5.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:traverse -s 4 -c 1 -o $O/f_cfg5 -f $Q > $O/f_ncu5.log 2>&1
$Q --config 4 > $O/f_q4.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:traverse -s 4 -c 1 -o $O/f_cfg4 -f $Q --config 4 > $O/f_ncu4.log 2>&1
# configs 1-3: the four phases of the second call, L2 / DRAM / efficiency metrics
for k in 1 2 3; do
  $Q --config $k > $O/f_q$k.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum.per_second,lts__t_bytes.sum,dram__bytes.sum.per_second,dram__bytes.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__cycles_elapsed.avg \
      --clock-control none -k regex:traverse -s 4 -c 4 --csv --log-file $O/f_metrics_cfg$k.csv $Q --config $k > $O/f_ncu_cfg$k.log 2>&1
done
for k in 5 4; do ncu -i $O/f_cfg$k.ncu-rep --page raw --csv > $O/f_cfg${k}_raw.csv 2>/dev/null; done
echo profile-done
