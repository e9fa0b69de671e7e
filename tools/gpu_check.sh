#!/bin/bash
# One GPU round-trip: parity tests, per-phase profiles, bench.  Run under gpurun.
set -u
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for spec in "cfg2 1024" "cfg3 1024" "cfg1 64" "cfg1 1024"; do
  set -- $spec
  timeout 300 python tools/profile_decode.py --cfg $1 --frames $2 --reps 2 > gpurun_out/ph_$1_$2.json 2>&1
  python - "$1" "$2" <<'PY'
import json, sys
c, f = sys.argv[1], sys.argv[2]
try:
    d = json.load(open(f"gpurun_out/ph_{c}_{f}.json")); r = d["runs"][-1]
    rd = lambda v: [round(x, 3) for x in v] if isinstance(v, list) else v
    print(c, f, "iters", round(d["mean_iterations"], 3), "good", d["good"], "kernel_ms", round(r["kernel_ms"], 3),
          "check", rd(r.get("check_ms")), "var", rd(r.get("var_ms")), "syn", rd(r.get("syncheck_ms")))
except Exception as ex:
    print(c, f, "FAILED", ex, open(f"gpurun_out/ph_{c}_{f}.json").read()[-500:])
PY
done
if [ "${BENCH:-1}" = "1" ]; then
  timeout 400 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench_rc=$?"
  python -c "
import json; l=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print('bench value', l['value'], 'e2e', l['e2e']['value'], 'frac', l['roofline']['frac'], 'kernel_ms', l['roofline']['kernel_ms'], 'cpu', l.get('cpu_baseline',{}).get('value'), 'sweep', l.get('qber_sweep'))"
fi
