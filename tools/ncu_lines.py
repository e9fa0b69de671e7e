"""Per-CUDA-source-line warp-stall samples of an ncu report (needs -lineinfo
and --import-source on):  python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
res = []
fname = None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[2] != "-":   # cuda rows carry "-" in the SASS address column
        continue
    try:
        s = int(r[4] or 0)
        ie = int(r[7] or 0)
    except ValueError:
        continue
    res.append((s, fname, r[0], r[1].strip()[:100], ie))
tot = sum(x[0] for x in res) or 1
print(f"total samples {tot}")
for s, f, ln, src, ie in sorted(res, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {f:14s} {ln:>5} inst={ie:>10} {src}")


def line_table(rep):
    """[(file, line, samples, inst_executed)] for every CUDA source line."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fname, hdr = [], None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[2] != "-":
            continue
        try:
            rows.append((fname, int(r[0]), int(r[4] or 0), int(r[7] or 0)))
        except ValueError:
            pass
    return rows
