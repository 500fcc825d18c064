# quick check of the level passes: c2 + c4 bench, parity subset (or $1), ncu of the W-side kernels on c4
out=gpurun_out/wc; mkdir -p $out
for c in c2 c4; do timeout 300 python bench.py --config $c --quick --steps 10 --warmup 3 > $out/quick_$c.json 2> $out/quick_$c.err; echo "quick $c rc=$?"; cat $out/quick_$c.json; tail -2 $out/quick_$c.err; done
timeout 900 python -m pytest tests -m gpu -q -x -k "${1:-c2 or c4 or full or emulated or 512 or 3}" > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu.log
