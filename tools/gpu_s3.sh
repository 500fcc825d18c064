#!/bin/bash
# c3 quick bench, then the k_dst_lvl4 parity cases (level passes at 1023^2, full-size c3 vs device oracle)
set -u
out=gpurun_out/s3; mkdir -p $out
timeout -s KILL 100 python bench.py --quick --steps 20 --warmup 3 > $out/bench.json 2> $out/bench.err || { echo "bench failed rc=$?"; tail -5 $out/bench.err; exit 1; }
python -c "import json; d=json.load(open('$out/bench.json')); print(round(d['ms_per_step'],3), [round(v,3) for v in d['phases_ms'].values()])"
timeout -s KILL 300 python -m pytest tests/test_gpu_levels.py -x -q -m gpu -k "1024" 2>&1 | tail -3
if [ -n "${FULL:-}" ]; then timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "full_size or graph_replay" 2>&1 | tail -3; fi
