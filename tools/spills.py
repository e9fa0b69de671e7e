"""Spill (STL/LDL) instructions per source line of one kernel in an object:
    python tools/spills.py obj.o kernel_substring"""
import re
import subprocess
import sys
import tempfile
from collections import Counter
from pathlib import Path

obj, pat = sys.argv[1], sys.argv[2]
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=td, capture_output=True)
    cub = next(Path(td).glob("*.cubin"))
    sass = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True, text=True).stdout
cur = fn = None
c = Counter()
tot = Counter()
for l in sass.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        fn = m.group(1)
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if fn and pat in fn and re.match(r"\s*/\*[0-9a-f]+\*/", l):
        tot[fn] += 1
        if re.search(r"\b(STL|LDL)\b", l):
            c[cur] += 1
for k, v in c.most_common(25):
    print(k, v)
print(dict(tot))
