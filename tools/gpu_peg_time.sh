#!/bin/bash
set -u
for spec in "4096 2048 1 2" "16384 8192 1001" "65536 32768 1 2"; do
  timeout 900 python tools/peg_gpu_time.py $spec 2>&1 | tail -3
done
