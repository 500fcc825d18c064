#!/bin/bash
# L2 retention probe (tools/probe_l2.cu) under ncu WITHOUT its cache flush between
# kernels: DRAM reads of k_read = bytes of the freshly written buffer L2 lost.
set -u
out=gpurun_out/l2; mkdir -p $out
timeout 600 ncu --cache-control none --clock-control none -k regex:"k_read|k_write" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum ./tools/probe_l2 > $out/probe_ncu.log 2>&1
echo "probe rc=$?"
