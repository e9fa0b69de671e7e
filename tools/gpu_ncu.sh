#!/bin/bash
# One ncu --set full capture of the decode kernel (cfg/frames from env).  Run under gpurun.
set -u
CFG=${CFG:-cfg2}; FRAMES=${FRAMES:-1024}; KREGEX=${KREGEX:-decode_scatter}; TAG=${TAG:-sc}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$KREGEX -c 1 -f \
  -o gpurun_out/${TAG}_${CFG}_full python tools/profile_decode.py --cfg $CFG --frames $FRAMES --once \
  > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu_rc=$?"; tail -3 gpurun_out/ncu_${TAG}.log
