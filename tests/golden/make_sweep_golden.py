"""Golden rows for the GPU sweep backend (paper_2001_07979_b200/sweep.py),
produced by the REFERENCE's own bench.run_sweep / measure_throughput
(bench.py:133-242) on the cfg-1 ensemble.  Timing fields are dropped (they
are the only fields allowed to differ).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_sweep_golden.py
"""
import io
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(OUT))
sys.path.insert(0, "/root/reference/pkg/src")

from make_golden import meta, ref_ensemble  # noqa: E402
from mmrecon import bench  # noqa: E402  (reference)

KEEP = ("e", "u", "R", "f", "frames", "success_rate", "mean_iterations", "residual_error_rate")


def main():
    ens = ref_ensemble("cfg1_n4096_m2048_u2_s1.npz")
    spec = bench.SweepSpec(e_values=(0.03, 0.09, 0.2), u_values=(1, 2), ensembles={0.5: ens}, frames=24,
                           warmup=2, seed=3)
    sink = io.StringIO()
    rows = bench.run_sweep(spec, sink)
    header = [ln for ln in sink.getvalue().splitlines() if ln.startswith("#")] + \
             [sink.getvalue().splitlines()[len(bench.CSV_DOC_LINES)]]
    points = {}
    for name, kw in (("prior", dict(prior_e=0.05)), ("calibrate", dict(calibrate=True))):
        p = bench.measure_throughput(ens, 2, 0.07, frames=20, seed=4, warmup=1, point_path=(5,), **kw)
        points[name] = {k: getattr(p, k) for k in ("mean_iterations", "iterations_std", "success_rate",
                                                   "residual_error_rate", "frames")}
    out = {"rows": [{k: getattr(r, k) for k in KEEP} for r in rows], "csv_header": header,
           "points": points, "meta": meta()}
    (OUT / "golden_sweep.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out["rows"], indent=0)[:600])


if __name__ == "__main__":
    main()
