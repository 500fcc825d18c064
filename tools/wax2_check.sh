# quick A/B of the W pass variant $1 on c2: bench, parity subset, ncu capture
V=${1:-4}; out=gpurun_out/w$V; mkdir -p $out
export BHCP_WAX_VARIANT=$V
timeout 300 python bench.py --quick --steps 30 --warmup 5 > $out/quick.json 2> $out/quick.err; echo "quick rc=$?"; cat $out/quick.json; tail -3 $out/quick.err
timeout 600 python -m pytest tests -m gpu -q -x -k "c2 or full or emulated or 512" > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu.log
ncu --set full --clock-control none --import-source on -k regex:"k_dst_wax" -s 1 -c 1 -o $out/wax -f python tools/profile_step.py c2 1 > $out/ncu.log 2>&1; echo "ncu rc=$?"
