"""Instructions executed / stall samples per device function of scatter.cuh
(line ranges found by scanning the source):  python tools/ncu_funcs.py rep"""
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
src = (Path(__file__).resolve().parents[1] / "paper_2001_07979_b200/csrc/scatter.cuh").read_text().splitlines()
starts = []
for i, l in enumerate(src, 1):
    m = re.match(r"\s*(?:static\s+)?(?:__device__|__global__).*?\b(\w+)\s*\(", l)
    if m:
        starts.append((i, m.group(1)))
    m = re.match(r"(\w+)\(const ScatterArgs A\)", l)
    if m:
        starts.append((i, m.group(1)))
starts.sort()


def func_of(line):
    name = "header"
    for s, n in starts:
        if s <= line + 3:   # template<> lines precede the signature
            name = n
    return name


exec(open(Path(__file__).resolve().parent / "ncu_lines.py").read().split("rep = sys.argv[1]")[0])
code = open(Path(__file__).resolve().parent / "ncu_lines.py").read()
ns = {}
exec(code[code.index("def line_table"):], {"subprocess": __import__("subprocess"), "csv": __import__("csv"),
                                           "io": __import__("io")}, ns)
rows = ns["line_table"](sys.argv[1])
agg = {}
for f, l, s, i in rows:
    key = func_of(l) if f == "scatter.cuh" else f
    a = agg.setdefault(key, [0, 0])
    a[0] += s
    a[1] += i
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} samples {100 * v[0] / ts:5.1f}%  inst {v[1] / 1e6:8.1f}M ({100 * v[1] / ti:4.1f}%)")
print(f"total inst {ti / 1e6:.1f}M")
