#!/bin/bash
# bench at N=1 (default flags) and N=2 (self-launched ranks sharing the GPU)
set -u
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench1.log 2>&1; echo "bench1 rc=$?"; tail -c 3000 gpurun_out/bench1.log
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --no-sweep > gpurun_out/bench2.log 2>&1; echo "bench2 rc=$?"; tail -c 1500 gpurun_out/bench2.log
