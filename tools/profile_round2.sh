#!/bin/bash
# Round-2 ncu evidence (run on the GPU box via gpurun; one GPU, one process).
# Each profiled command first runs once without ncu and must exit 0.
O=gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu"
Q="python bench.py --steps 1 --warmup 3 --no-cpu --quick"
$B > $O/p2_plain.json 2> $O/p2_plain.err && \
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum --clock-control none \
      --csv --log-file $O/p2_launches_cfg5.csv $B > $O/p2_ncu_list.log 2>&1
$Q > $O/p2_q5.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:traverse -s 4 -c 1 -o $O/p2_cfg5 -f $Q > $O/p2_ncu5.log 2>&1
$Q --config 4 > $O/p2_q4.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:traverse -s 4 -c 1 -o $O/p2_cfg4 -f $Q --config 4 > $O/p2_ncu4.log 2>&1
for k in 1 2 3; do
  $Q --config $k > $O/p2_q$k.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum.per_second,lts__t_bytes.sum,dram__bytes.sum.per_second,dram__bytes.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__cycles_elapsed.avg \
      --clock-control none -k regex:traverse -s 4 -c 4 --csv --log-file $O/p2_metrics_cfg$k.csv $Q --config $k > $O/p2_ncu_cfg$k.log 2>&1
done
for k in 5 4; do ncu -i $O/p2_cfg$k.ncu-rep --page raw --csv > $O/p2_cfg${k}_raw.csv 2>/dev/null; done
echo profile-done
