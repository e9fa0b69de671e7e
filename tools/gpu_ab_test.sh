#!/bin/bash
# A/B one variant library against the in-tree one (per-phase profiles of
# cfg2/cfg3), then the GPU parity tests on the variant.  Run under gpurun:
#   bash tools/gpu_ab_test.sh gpurun_libs/<name>/libmbp_b200.so
set -u
mkdir -p gpurun_out
bash tools/ab_libs.sh "$@" 2>&1 | tee gpurun_out/ab.log
for lib in "$@"; do
  MBP_LIB=$lib timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/ab_pytest.log 2>&1
  echo "pytest $lib rc=$?"; tail -3 gpurun_out/ab_pytest.log
done
