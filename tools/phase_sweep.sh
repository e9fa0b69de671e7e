#!/bin/bash
# Per-phase decode times for several batch sizes (cfg and sizes from args).
CFG=${1:-cfg2}; shift
for f in "${@:-128 1024}"; do
  timeout 300 python tools/profile_decode.py --cfg $CFG --frames $f --reps 3 > gpurun_out/ps.json 2>&1
  python - "$CFG" "$f" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ps.json")); r = d["runs"][-1]
rd = lambda v: [round(x, 3) for x in v] if isinstance(v, list) else v
print(sys.argv[1], sys.argv[2], "kernel", round(r["kernel_ms"], 3), "syn0", round(r["syncheck0_ms"], 3), "check", rd(r.get("check_ms")),
      "var", rd(r.get("var_ms")), "syn", rd(r.get("syncheck_ms")), "tail", round(r["tail_ms"], 3), "cmp", r.get("compaction_ms"))
PY
done
