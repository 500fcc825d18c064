#!/bin/bash
# Round-2 evidence on one B200: GPU tests, smoke, bench (c3 headline, c2 line,
# reference arm), all configs + CPU reference, the c5 batched sweep, ncu launch
# list of the c3 step and --set full captures of the step kernels of c3, c2,
# c4, c5 and c1. Usage (under gpurun): bash tools/evidence_r02.sh <tag>
set -u
tag=${1:-r02}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $out/rc.txt
tail -3 $out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $out/rc.txt
python bench.py > $out/bench_c3.json 2> $out/bench_c3.err; echo "bench rc=$?" | tee -a $out/rc.txt
head -c 1500 $out/bench_c3.json; echo
python bench.py --config c2 > $out/bench_c2.json 2> $out/bench_c2.err; echo "bench c2 rc=$?" | tee -a $out/rc.txt
python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?" | tee -a $out/rc.txt
python tools/sweep_c5.py > $out/sweep_c5.json 2> $out/sweep_c5.err; echo "sweep c5 rc=$?" | tee -a $out/rc.txt
python tools/run_configs.py --cpu > $out/configs.json 2> $out/configs.err; echo "configs rc=$?" | tee -a $out/rc.txt
python bench.py --quick --steps 3 --warmup 3 > $out/bench_short.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_c3.csv \
      python bench.py --quick --steps 3 --warmup 3 > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" | tee -a $out/rc.txt
# --set full captures, summarised on the box (the reports themselves exceed what
# gpurun copies back): raw metrics CSV, summary table, DRAM traffic, hot source lines
for cfg in c3 c2 c4 c5 c1; do
  python tools/profile_step.py $cfg 1 > $out/profile_step_$cfg.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -c 14 \
        -o /tmp/${cfg}_full -f python tools/profile_step.py $cfg 1 > $out/ncu_full_$cfg.log 2>&1
  echo "ncu full $cfg rc=$?" | tee -a $out/rc.txt
  lf=-; [ "$cfg" = c3 ] && lf=$out/launches_c3.csv
  python tools/ncu_summary.py /tmp/${cfg}_full.ncu-rep $lf $out/r02_$cfg > /dev/null 2>&1
  python tools/src_hot.py /tmp/${cfg}_full.ncu-rep 40 > $out/r02_${cfg}_src_hot.txt 2>&1
  rm -f /tmp/${cfg}_full.ncu-rep
done
