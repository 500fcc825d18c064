#!/bin/bash
# A/B timing of library variants under tools/_abl/ on one box (quick bench of $CFG, twice each, interleaved)
for rep in 1 2; do
for v in tools/_abl/*.so; do
  cp $v paper_2107_06381_b200/libbhcp_b200.so
  timeout -s KILL 200 python bench.py --quick --config ${CFG:-c3} --steps ${STEPS:-20} --warmup 3 > /tmp/b.json 2>/tmp/b.err || { echo "$v failed"; tail -3 /tmp/b.err; continue; }
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$v', round(d['ms_per_step'],3), [round(v,3) for v in d['phases_ms'].values()])"
done
done
