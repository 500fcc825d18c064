#!/bin/bash
# Round evidence on one B200: tests, bench (both arms), all configs, ncu launch
# list of the bench command, one --set full capture of the three step kernels.
# Usage (under gpurun): bash tools/evidence.sh <tag>
set -u
tag=${1:-r01}
out=gpurun_out/$tag
mkdir -p $out
python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $out/rc.txt
python bench.py > $out/bench_c2.json 2> $out/bench_c2.err; echo "bench rc=$?" | tee -a $out/rc.txt
python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?" | tee -a $out/rc.txt
python tools/run_configs.py --cpu > $out/configs.json 2> $out/configs.err; echo "configs rc=$?" | tee -a $out/rc.txt
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
./tools/probe_fp64 > $out/probe_fp64.txt 2>&1; echo "probe_fp64 rc=$?" | tee -a $out/rc.txt
tail -3 $out/pytest_gpu.log
cat $out/bench_c2.json | head -c 3000
