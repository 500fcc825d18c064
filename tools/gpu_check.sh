#!/bin/bash
# full GPU suite + smoke + c3 bench (quick) on one B200: bash tools/gpu_check.sh <tag>
set -u
tag=${1:-chk}
out=gpurun_out/$tag; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 $out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $out/bench_c3.json 2> $out/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('$out/bench_c3.json')); print(round(d['ms_per_step'],3), d['value']/1e9, [round(v,3) for v in d['phases_ms'].values()], d['e2e']['value']/1e9)" 2>&1 | tail -1
