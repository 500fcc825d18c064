# c3 pass A rewrite: parity subset, c3 timing, ncu of the new kernel
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g2_smoke.log 2>&1; echo smoke_rc=$?
tail -12 gpurun_out/g2_smoke.log
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "1024 or 1025 or c3 or graph or distributed or residue" > gpurun_out/g2_tests.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/g2_tests.log
python bench.py --quick --steps 10 --warmup 3 > gpurun_out/g2_c3q.json 2>&1; echo c3q=$?
cat gpurun_out/g2_c3q.json
timeout 600 ncu --set full --import-source on -k regex:k_modes_gt -c 1 -o gpurun_out/g2_gt python bench.py --quick --steps 1 --warmup 1 > gpurun_out/g2_ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/g2_ncu.log
