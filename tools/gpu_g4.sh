timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "1024 or 1025 or c3 or graph or distributed or residue or smallest or singular" > gpurun_out/g4_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/g4_tests.log
for i in 1 2; do python bench.py --quick --steps 10 --warmup 3; done > gpurun_out/g4_c3q.json 2>&1; echo c3q=$?
cat gpurun_out/g4_c3q.json
timeout 600 ncu --set full --import-source on -k regex:k_modes_gt -c 1 -o gpurun_out/g4_gt python bench.py --quick --steps 1 --warmup 1 > gpurun_out/g4_ncu.log 2>&1; echo ncu=$?
