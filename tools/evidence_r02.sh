#!/bin/bash
# Round-2 evidence on one B200: GPU tests, smoke, bench (c3 headline, c2 line,
# reference arm), ncu launch list of the c3 step and one --set full capture of
# every c3 step kernel. Usage (under gpurun): bash tools/evidence_r02.sh <tag>
set -u
tag=${1:-r02}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
python -m pytest tests -m gpu -q -x -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $out/rc.txt
tail -3 $out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $out/rc.txt
python bench.py > $out/bench_c3.json 2> $out/bench_c3.err; echo "bench rc=$?" | tee -a $out/rc.txt
cat $out/bench_c3.json | head -c 4000; echo
python bench.py --config c2 > $out/bench_c2.json 2> $out/bench_c2.err; echo "bench c2 rc=$?" | tee -a $out/rc.txt
python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?" | tee -a $out/rc.txt
python bench.py --quick --steps 3 --warmup 3 > $out/bench_short.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_c3.csv \
      python bench.py --quick --steps 3 --warmup 3 > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" | tee -a $out/rc.txt
python tools/profile_step.py c3 1 > $out/profile_step.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -c 12 \
      -o $out/c3_full -f python tools/profile_step.py c3 1 > $out/ncu_full.log 2>&1; echo "ncu full rc=$?" | tee -a $out/rc.txt
