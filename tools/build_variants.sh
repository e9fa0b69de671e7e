#!/bin/bash
# Build A/B variants of libmbp_b200.so under gpurun_libs/<name>/ (CPU; nvcc cross-compiles)
set -u
cd /root/repo
build() {  # name define...
  name=$1; shift
  python - "$name" "$@" <<'PY'
import sys
from paper_2001_07979_b200.build import build
name, defs = sys.argv[1], sys.argv[2:]
build(force=True, defines=defs, out=f"/root/repo/gpurun_libs/{name}/libmbp_b200.so")
print("built", name, defs, flush=True)
PY
}
for spec in "$@"; do
  build $spec
done
