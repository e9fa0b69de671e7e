#!/bin/bash
# A/B of library variants: per-phase profile of cfg2/cfg3 (1024 frames) with
# the default library and each variant given as an argument (a .so path).
# Run under gpurun.
set -u
summ() {
python - "$1" <<'PY'
import json, sys
d = json.load(open(sys.argv[1])); r = d["runs"][-1]
rd = lambda v: [round(x, 3) for x in v] if isinstance(v, list) else v
print("  iters", round(d["mean_iterations"], 3), "good", d["good"], "kernel_ms", round(r["kernel_ms"], 3),
      "check", rd(r.get("check_ms")), "var", rd(r.get("var_ms")), "syn", rd(r.get("syncheck_ms")), "cmp", r.get("compaction_ms", {}).get("move"))
PY
}
for lib in default "$@"; do
  echo "== $lib"
  for cfg in cfg2 cfg3; do
    if [ "$lib" = default ]; then
      timeout 300 python tools/profile_decode.py --cfg $cfg --frames 1024 --reps 3 > gpurun_out/ab.json 2>&1
    else
      MBP_LIB=$lib timeout 300 python tools/profile_decode.py --cfg $cfg --frames 1024 --reps 3 > gpurun_out/ab.json 2>&1
    fi
    echo " $cfg"; summ gpurun_out/ab.json || tail -5 gpurun_out/ab.json
  done
done
