#!/bin/bash
# ncu --set full of k_dst_lvl4 (one launch) + stall shares
set -u
out=gpurun_out/s4; mkdir -p $out
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:k_dst_lvl4 -s 1 -c 1 -o $out/lvl4 -f python tools/profile_step.py c3 1 > $out/ncu.log 2>&1
python tools/ncu_brief.py $out/lvl4.ncu-rep
