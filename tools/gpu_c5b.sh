#!/bin/bash
# c5 pass A check: 4097-level parity tests (incl. singular shifts), pass-A timing, sweep
set -u
out=gpurun_out/c5b; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "4097 or 4096 or sweep or batched or c5 or singular" > $out/tests.log 2>&1; echo "tests rc=$?"
tail -1 $out/tests.log
timeout 300 python bench.py --config c5 --quick --steps 20 --warmup 3 > $out/bench.json 2>&1
python -c "import json; d=json.load(open('$out/bench.json')); print(round(d['ms_per_step'],4), [round(v,4) for v in d['phases_ms'].values()])" 2>&1 | tail -1
timeout 600 python tools/sweep_c5.py > $out/sweep.json 2>&1; python -c "import json; d=json.load(open('$out/sweep.json')); print(d['runs'][-1], d['max_rel_dev_e_h'])"
python tools/profile_step.py c5 1 > /dev/null; timeout 600 ncu --clock-control none -k regex:k_modes_pf -c 1 --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__t_sector_hit_rate.pct python tools/profile_step.py c5 1 2>&1 | grep -E "    [a-z]"
