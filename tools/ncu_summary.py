"""Summarise an ncu report (one kernel launch) into profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_decode_ncu.md [--traffic-json profiles/decode_traffic.json --frames 1024 --e 0.03]
"""
import argparse
import csv
import io
import json
import subprocess
from collections import Counter

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def opmix(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    c = Counter()
    stalls = Counter()
    for r in rows[2:]:
        toks = r[ix["Source"]].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        try:
            c[op] += float(r[ix["Instructions Executed"]])
        except ValueError:
            pass
        for h in hdr:
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    stalls[h] += float(r[ix[h]])
                except ValueError:
                    pass
    return c, stalls


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--traffic-json")
    ap.add_argument("--frames", type=int, default=1024)
    ap.add_argument("--e", type=float, default=0.03)
    ap.add_argument("--title", default="decode_kernel")
    ap.add_argument("--workload", default="cfg2")
    a = ap.parse_args()
    m = raw(a.rep)
    lines = [f"# ncu summary: {a.title}", "", f"report: `{a.rep}` (ncu --set full --clock-control none)", "",
             "| metric | value | unit |", "|---|---|---|"]
    name = m.get("Kernel Name", ("?", ""))[0]
    lines.insert(2, f"kernel: `{name}`")
    for k in KEYS:
        if k in m:
            lines.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
    ops, stalls = opmix(a.rep)
    tot = sum(ops.values()) or 1
    lines += ["", "## executed instruction mix (warp-level)", "", "| op | share |", "|---|---|"]
    for op, v in ops.most_common(16):
        lines.append(f"| {op} | {100 * v / tot:.1f}% |")
    st = sum(stalls.values()) or 1
    lines += ["", "## warp stall samples", "", "| reason | share |", "|---|---|"]
    for s, v in stalls.most_common(10):
        lines.append(f"| {s} | {100 * v / st:.1f}% |")
    open(a.out, "w").write("\n".join(lines) + "\n")

    def num(k):
        v, u = m[k]
        v = float(v.replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
        return v * scale
    if a.traffic_json and "dram__bytes_read.sum" in m:
        # one record per (workload, frames, e), keyed to the library sources
        # the capture ran on (bench.py drops `traffic` for other sources)
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        from paper_2001_07979_b200.build import source_hash

        t = {"workload": a.workload, "frames": a.frames, "e": a.e, "src_sha": source_hash(),
             "dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
             "dram_read": num("dram__bytes_read.sum"), "dram_write": num("dram__bytes_write.sum"),
             "kernel_ms_ncu": num("gpu__time_duration.sum") / (1e6 if m["gpu__time_duration.sum"][1] == "ns" else 1e3
                                                               if m["gpu__time_duration.sum"][1] == "us" else 1),
             "capture": Path(a.rep).name, "summary": a.out}
        try:
            old = json.loads(open(a.traffic_json).read())
            old = old if isinstance(old, list) else [old]
        except (OSError, ValueError):
            old = []
        keep = [r for r in old if (r.get("workload"), r.get("frames"), r.get("e")) != (a.workload, a.frames, a.e)]
        open(a.traffic_json, "w").write(json.dumps(keep + [t], indent=1) + "\n")
    print("\n".join(lines[:30]))


if __name__ == "__main__":
    main()
