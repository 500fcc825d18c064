#!/bin/bash
# k_dst_lvl4 consumer layout / ping-pong modes: c3 quick bench per BHCP_LVL4_MODE, then parity of the chosen one
set -u
out=gpurun_out/s2; mkdir -p $out
for md in ${MODES:-0 1 2}; do
  BHCP_LVL4_MODE=$md timeout 200 python bench.py --quick --steps 20 --warmup 3 > $out/bench_m$md.json 2> $out/bench_m$md.err || { echo "mode $md failed rc=$?"; tail -3 $out/bench_m$md.err; continue; }
  python -c "import json; d=json.load(open('$out/bench_m$md.json')); print('mode $md', round(d['ms_per_step'],3), [round(v,3) for v in d['phases_ms'].values()])"
done
if [ -n "${PARITY:-}" ]; then
  BHCP_LVL4_MODE=$PARITY timeout 900 python -m pytest tests/test_gpu_levels.py tests/test_gpu_parity.py -x -q -m gpu -k "${KEXPR:-1023 or lvl4 or c3 or full_size}" 2>&1 | tail -5
fi
