#!/bin/bash
# ncu --set full of one kernel of one config: bash tools/gpu_s5.sh <config> <kernel-regex>
set -u
cfg=${1:-c4}; k=${2:-k_modes_rader}
out=gpurun_out/s5; mkdir -p $out
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o $out/${cfg}_$k -f python tools/profile_step.py $cfg 1 > $out/ncu_${cfg}_$k.log 2>&1
python tools/ncu_brief.py $out/${cfg}_$k.ncu-rep
python tools/sass_hot.py $out/${cfg}_$k.ncu-rep "" 25
python tools/src_hot.py $out/${cfg}_$k.ncu-rep 25 2>/dev/null | head -30
