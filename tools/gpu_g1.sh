set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/g1_tests.log 2>&1; echo tests_rc=$?
tail -30 gpurun_out/g1_tests.log
python bench.py --config c2 --quick --steps 50 --warmup 5 > gpurun_out/g1_c2q.json 2>gpurun_out/g1_c2q.err; echo c2q=$?
python bench.py --steps 10 --warmup 3 > gpurun_out/g1_c3.json 2>gpurun_out/g1_c3.err; echo c3=$?
cat gpurun_out/g1_c2q.json; head -c 1500 gpurun_out/g1_c3.json
