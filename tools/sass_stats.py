"""Per-kernel SASS statistics from cuobjdump (instruction mix of one function)."""
import re
import subprocess
import sys
from collections import Counter

lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if not re.search(pat, name):
        continue
    ops = Counter()
    n = 0
    for line in f.split("\n"):
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            ops[m.group(2).split(".")[0]] += 1
            n += 1
    print(name, "instructions:", n)
    print("  ", ", ".join(f"{k}:{v}" for k, v in ops.most_common(25)))
