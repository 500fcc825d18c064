#!/bin/bash
for v in tools/_abl/*.so; do
cp $v paper_2107_06381_b200/libbhcp_b200.so
echo $v
timeout -s KILL 100 python tools/profile_step.py c3 0 2>&1 | tail -3
done
