#!/bin/bash
# A/B of a runtime switch (env var $AB, e.g. MBP_NO_HOT=1) on the bench
# workloads: cfg2 (e = 0.03, 0.05) and cfg3, alternating runs.  Under gpurun.
set -u
TAG=${TAG:-ab}
AB=${AB:-MBP_NO_HOT=1}
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest_gpu.log
fi
for rep in 1 2; do
  for we in cfg2:0.03 cfg3:0.03 cfg2:0.05; do
    w=${we%%:*}; e=${we##*:}
    for mode in B A; do
      if [ $mode = A ]; then envs="env $AB"; else envs="env"; fi
      $envs timeout 300 python bench.py --workload $w --e $e --steps 20 --warmup 5 --no-sweep --no-extra --stream 0 --no-cpu-baseline > gpurun_out/${TAG}_${w}_${e}_${mode}${rep}.log 2>&1
      python - "$w$e" "$mode" gpurun_out/${TAG}_${w}_${e}_${mode}${rep}.log <<'PY'
import json, sys
w, mode, f = sys.argv[1:]
ls = [l for l in open(f) if l.startswith('{')]
if not ls: print(w, mode, 'no line'); sys.exit()
d = json.loads(ls[-1])
print(w, mode, d['value'], 'kernel_ms', d['roofline'].get('kernel_ms'), 'step', d['ms_per_step'], 'e2e', d['e2e']['value'])
PY
    done
  done
done
