mkdir -p gpurun_out/ab
for V in 0 1 2 3; do BHCP_WAX_VARIANT=$V python bench.py --quick --steps 30 --warmup 5 > gpurun_out/ab/c2_v$V.json 2>&1; echo "c2 v$V"; cat gpurun_out/ab/c2_v$V.json | tail -1; done
for V in 0 1; do BHCP_WAX_VARIANT=$V python bench.py --config c3 --quick --steps 5 --warmup 3 > gpurun_out/ab/c3_v$V.json 2>&1; echo "c3 v$V"; tail -1 gpurun_out/ab/c3_v$V.json; done
for V in 0 1; do BHCP_WAX_VARIANT=$V timeout 300 python bench.py --config c4 --quick --steps 3 --warmup 3 > gpurun_out/ab/c4_v$V.json 2>&1; echo "c4 v$V"; tail -1 gpurun_out/ab/c4_v$V.json; done
