#!/bin/bash
# ncu part of tools/evidence.sh only. Usage: bash tools/evidence_ncu.sh <tag>
set -u
tag=${1:-r01}
out=gpurun_out/$tag
mkdir -p $out
# launch list of the timed step (--quick: device step only) and of the whole bench command
python bench.py --quick --steps 3 --warmup 3 > $out/bench_short.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
      python bench.py --quick --steps 3 --warmup 3 > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" | tee -a $out/rc.txt
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_short_full.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_full_bench.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $out/ncu_launch_full.log 2>&1; echo "ncu launches full rc=$?" | tee -a $out/rc.txt
python tools/profile_step.py c2 1 > $out/profile_step.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_dst_blk3|k_modes_fast|k_dst_wax2" -s 3 -c 3 \
      -o $out/c2_full -f python tools/profile_step.py c2 2 > $out/ncu_full.log 2>&1; echo "ncu full rc=$?" | tee -a $out/rc.txt
