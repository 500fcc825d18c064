#!/bin/bash
# quick check: device bench + a few ncu metrics for the given kernel regex.
# usage: bash tools/quick_ncu.sh <kernel-regex> [config]
set -u
cfg=${2:-c2}
python bench.py --quick --config $cfg --steps 20 --warmup 5 || exit 1
python tools/profile_step.py $cfg 1 > /dev/null || exit 1
ncu --clock-control none -k regex:"$1" -s 1 -c 2 --metrics \
gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  python tools/profile_step.py $cfg 1 2>&1 | grep -E "k_|duration|wavefronts|conflicts|throughput|warps_active|inst_executed|dram__bytes" 
