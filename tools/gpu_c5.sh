#!/bin/bash
# c5 batched sweep: parity tests + timing of the full 128-solve sweep (device + wall)
set -u
out=gpurun_out/c5; mkdir -p $out
timeout 900 python -m pytest tests/test_sweep.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "sweep or batched or c5" > $out/tests.log 2>&1; echo "tests rc=$?"
tail -2 $out/tests.log
timeout 900 python tools/sweep_c5.py > $out/sweep.json 2> $out/sweep.err; echo "sweep rc=$?"
tail -c 1500 $out/sweep.json; tail -3 $out/sweep.err
