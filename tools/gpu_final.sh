#!/bin/bash
# End-of-round measurement on one B200 (run under gpurun): tests, bench lines,
# launch list, full ncu capture of the decode kernel, sanitizers.
set -u
TAG=${TAG:-r02b}
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest_gpu.log
fi
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --no-sweep --no-extra > gpurun_out/${TAG}_bench_gpus2.log 2>&1; echo "bench2 rc=$?"
for w in cfg3 cfg1 cfg4; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-sweep --no-extra --stream 0 > gpurun_out/${TAG}_bench_$w.log 2>&1; echo "bench $w rc=$?"
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${TAG}_bench_reference.log 2>&1; echo "reference rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep --no-extra --stream 0 > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_scatter -c 1 -f \
  -o gpurun_out/${TAG}_cfg2_full python tools/profile_decode.py --cfg cfg2 --frames 1024 --once > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:decode_scatter -c 2 --csv --log-file gpurun_out/${TAG}_dram_cfg3.csv \
  python tools/profile_decode.py --cfg cfg3 --frames 1024 --once > /dev/null 2>&1; echo "ncu cfg3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:decode_scatter -c 1 --csv --log-file gpurun_out/${TAG}_dram_cfg4.csv \
  python tools/profile_decode.py --cfg cfg4 --frames 1024 --once > /dev/null 2>&1; echo "ncu cfg4 rc=$?"
if [ "${SAN:-1}" = "1" ]; then
  timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/${TAG}_san_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -2 gpurun_out/${TAG}_san_memcheck.log
fi
