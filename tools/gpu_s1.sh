#!/bin/bash
# session check: c3 quick bench, ncu --set full of k_dst_lvl4 and k_modes_gt with stall shares
set -u
out=gpurun_out/s1; mkdir -p $out
timeout 300 python bench.py --quick --steps 20 --warmup 3 > $out/bench_c3.json 2> $out/bench_c3.err
python -c "import json; d=json.load(open('$out/bench_c3.json')); print(round(d['ms_per_step'],3), d['phases_ms'])"
for k in k_dst_lvl4 k_modes_gt; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o $out/$k -f python tools/profile_step.py c3 1 > $out/ncu_$k.log 2>&1
  python tools/ncu_brief.py $out/$k.ncu-rep > $out/brief_$k.txt 2>&1
  cat $out/brief_$k.txt
done
