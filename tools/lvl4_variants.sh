#!/bin/bash
# k_dst_lvl4 look-ahead sweep: c3 device bench + ncu DRAM bytes per BHCP_LVL4_KFIRST
# (row-task pairs of a phase before the column tasks; default = grid size)
set -u
out=gpurun_out/lvl4v; mkdir -p $out
run() {
  n=$1; shift
  env "$@" timeout 300 python bench.py --quick --steps 20 --warmup 3 > $out/bench_$n.json 2>&1
  python -c "import json; d=json.load(open('$out/bench_$n.json')); print('$n', round(d['ms_per_step'],3), [round(v,3) for v in d['phases_ms'].values()])" 2>&1 | tail -1
  env "$@" timeout 300 ncu --clock-control none -k regex:k_dst_lvl4 -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct python tools/profile_step.py c3 1 > $out/ncu_$n.log 2>&1
  grep -E "duration|dram__|hit_rate" $out/ncu_$n.log | awk '{printf "  %s %s %s", $1, $2, $3} END {print ""}'
}
run k74 BHCP_LVL4_KFIRST=74
run k148 BHCP_LVL4_KFIRST=148
run k222 BHCP_LVL4_KFIRST=222
run blk4_cols3 BHCP_LVL4=0
