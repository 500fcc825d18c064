#!/bin/bash
# timing-only ablations of k_dst_lvl4 (results are wrong by construction)
for v in tools/_abl/*.so; do
  cp $v paper_2107_06381_b200/libbhcp_b200.so
  timeout -s KILL 100 python bench.py --quick --steps 10 --warmup 3 > /tmp/b.json 2>/tmp/b.err || { echo "$v failed"; tail -3 /tmp/b.err; continue; }
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$v', round(d['ms_per_step'],3), [round(v,3) for v in d['phases_ms'].values()])"
done
