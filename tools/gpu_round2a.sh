#!/bin/bash
# Round-2 first GPU call: tests, bench, sanitizers.  Run under gpurun.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench_rc=$?"; tail -c 600 gpurun_out/bench.log
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/san_$tool.log
done
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 50 python tools/sanitize_run.py --quick > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/san_racecheck.log
