#!/bin/bash
# bench N=1 / N=2, launch list, full ncu capture of the decode kernel (cfg2 1024 e=0.03)
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02a}
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench1.log 2>&1; echo "bench1 rc=$?"
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --no-sweep --no-extra > gpurun_out/bench2.log 2>&1; echo "bench2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep --no-extra --stream 0 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_scatter -c 1 -f \
  -o gpurun_out/${TAG}_cfg2_full python tools/profile_decode.py --cfg cfg2 --frames 1024 --once > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log
