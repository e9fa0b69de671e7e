#!/bin/bash
# decode-kernel time vs frames per launch (cfg2 e=0.03/0.05, cfg3 e=0.03)
set -u
for spec in "cfg2 0.03" "cfg2 0.05" "cfg3 0.03"; do
  set -- $spec
  for F in 1024 2048 4096 8192; do
    timeout 300 python tools/profile_decode.py --cfg $1 --e $2 --frames $F --reps 3 > gpurun_out/bs_$1_$2_$F.json 2>&1
    python - "$1" "$2" "$F" <<'PY'
import json, sys
c, e, f = sys.argv[1:4]
try:
    d = json.load(open(f"gpurun_out/bs_{c}_{e}_{f}.json")); r = d["runs"][-1]
    rd = lambda v: [round(x, 3) for x in v] if isinstance(v, list) else v
    ms = min(x["kernel_ms"] for x in d["runs"])
    print(c, e, f, "iters", round(d["mean_iterations"], 3), "good", d["good"], "kernel_ms", round(ms, 3),
          "per1024", round(ms * 1024 / int(f), 3), "check", rd(r.get("check_ms")), "var", rd(r.get("var_ms")),
          "syn", rd(r.get("syncheck_ms")), "cmp", r.get("compaction_ms"), flush=True)
except Exception as ex:
    print(c, e, f, "FAILED", ex, open(f"gpurun_out/bs_{c}_{e}_{f}.json").read()[-400:])
PY
  done
done
