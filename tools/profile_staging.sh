#!/bin/bash
# a3 A/B with ncu: treelet blocks staged in shared memory vs per-lane loads of
# the same aligned blobs (generic kernel both times), config 5, phase 0 of the
# second call: L1 wavefronts and requests per decoded record.
O=gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors.sum,l1tex__t_sector_hit_rate.pct,smsp__inst_executed_op_ldgsts.sum
for st in off on; do
  Q="python bench.py --steps 1 --warmup 3 --no-cpu --quick --align-treelets --staging $st"
  CBVH_FAST=0 $Q > $O/st_$st.json 2>&1 && \
  CBVH_FAST=0 ncu --metrics $M --clock-control none -k regex:traverse -s 4 -c 1 --csv --log-file $O/st_$st.csv $Q > $O/st_ncu_$st.log 2>&1
done
echo staging-profile-done
