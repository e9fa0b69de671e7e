#!/bin/bash
set -u
mkdir -p gpurun_out
bash tools/ab_libs.sh gpurun_libs/magic/libmbp_b200.so 2>&1 | tee gpurun_out/ab_magic.log
for spec in "4096 2048 1 2" "16384 8192 1001" "65536 32768 1"; do
  timeout 900 python tools/peg_gpu_time.py $spec 2>&1 | tail -3
done
