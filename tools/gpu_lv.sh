#!/bin/bash
# k_dst_lvl4 quick check: level parity tests, c3 quick bench, ncu DRAM, per-role cycle accounting
set -u
out=gpurun_out/lv; mkdir -p $out
for L in 9 23; do timeout 120 python tools/lvl4_debug.py $L; done
timeout 600 python -m pytest tests/test_gpu_levels.py -q -x -p no:cacheprovider > $out/tests_levels.log 2>&1; echo "levels rc=$?"
tail -1 $out/tests_levels.log
timeout 300 python bench.py --quick --steps 20 --warmup 3 > $out/bench.json 2>&1
python -c "import json; d=json.load(open('$out/bench.json')); print(round(d['ms_per_step'],3), [round(v,3) for v in d['phases_ms'].values()])" 2>&1 | tail -1
timeout 300 ncu --clock-control none -k regex:k_dst_lvl4 -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct python tools/profile_step.py c3 1 > $out/ncu.log 2>&1
grep -E "duration|dram__|hit_rate" $out/ncu.log | awk '{printf "  %s %s %s", $1, $2, $3} END {print ""}'
if [ -f paper_2107_06381_b200/libbhcp_b200_prof.so ]; then
  cp paper_2107_06381_b200/libbhcp_b200.so /tmp/keep.so; cp paper_2107_06381_b200/libbhcp_b200_prof.so paper_2107_06381_b200/libbhcp_b200.so
  timeout 300 python tools/profile_step.py c3 1 2>&1 | grep "cta 37" | tail -1
  cp /tmp/keep.so paper_2107_06381_b200/libbhcp_b200.so
fi
