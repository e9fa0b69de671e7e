"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into a
markdown table:  python tools/launch_table.py launches.csv out.md "title" """
import csv
import sys
from collections import defaultdict

src, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(src)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {h: i for i, h in enumerate(hdr)}
agg = defaultdict(list)
for r in rows[start + 1:]:
    if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
    agg[r[ix["Kernel Name"]]].append(v)
tot = sum(sum(v) for v in agg.values()) or 1
lines = [f"# {title}", "",
         "Cold-cache, serialised per-launch times (ncu); compare shares, not absolutes. "
         "`FillFunctor` = bench.py's L2 flush between timed steps (outside the timed region).", "",
         "| kernel | launches | total ms | mean ms | share |", "|---|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"| `{k[:80]}` | {len(v)} | {sum(v):.3f} | {sum(v) / len(v):.4f} | {100 * sum(v) / tot:.1f}% |")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
