#!/bin/bash
# LSU / shared-memory pipe counters of the two c3 step kernels (one launch each)
set -u
out=gpurun_out/s6; mkdir -p $out
for k in k_dst_lvl4 k_modes_gt; do
timeout -s KILL 300 ncu --clock-control none -k regex:$k -s 1 -c 1 --csv --metrics \
gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.max,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__inst_executed_pipe_lsu.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_global_st.sum,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed,l1tex__f_wavefronts.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum \
  python tools/profile_step.py c3 1 > $out/lsu_$k.csv 2> $out/lsu_$k.err
python - <<P
import csv
rows=[r for r in csv.reader(open('$out/lsu_$k.csv')) if len(r)>10]
h=rows[0]; 
for r in rows[1:]:
    print(r[h.index('Metric Name')], r[h.index('Metric Unit')], r[h.index('Metric Value')])
P
done
