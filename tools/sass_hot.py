"""Hot SASS regions of an ncu capture: per-instruction executed counts and
stall samples, grouped into basic-block-like runs of equal execution count.
    ncu -i rep --page source --csv --print-source sass > s.csv
    python tools/sass_hot.py s.csv [min_share]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
minshare = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ins = []
for r in rows[2:]:
    try:
        ins.append((r[ix["Address"]], r[ix["Source"]].strip(), float(r[ix["Instructions Executed"]] or 0),
                    float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
    except (ValueError, IndexError):
        pass
tot = sum(x[2] for x in ins)
stot = sum(x[3] for x in ins) or 1
# runs of equal execution count
runs = []
cur = None
for k, (a, s, n, st) in enumerate(ins):
    if cur and n == cur["n"]:
        cur["end"] = k
        cur["st"] += st
    else:
        cur = {"start": k, "end": k, "n": n, "st": st}
        runs.append(cur)
runs.sort(key=lambda r: -(r["n"] * (r["end"] - r["start"] + 1)))
print(f"total warp instructions {tot:.3e}, SASS lines {len(ins)}")
for r in runs[:40]:
    w = r["n"] * (r["end"] - r["start"] + 1)
    if w / tot < minshare:
        break
    print(f"{100 * w / tot:5.1f}% inst {100 * r['st'] / stot:5.1f}% stall  lines {r['start']}-{r['end']} "
          f"({r['end'] - r['start'] + 1} instr x {r['n']:.3e})  first: {ins[r['start']][1][:60]}")
