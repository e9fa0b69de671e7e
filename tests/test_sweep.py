"""GPU sweep backend (paper_2001_07979_b200/sweep.py) against the reference's
bench.run_sweep / measure_throughput (tests/golden/make_sweep_golden.py):
identical grid rows except the timing fields, CSV v1 byte-compatible."""

import io
import json
from pathlib import Path

import pytest

from paper_2001_07979_b200.sweep import (CSV_COLUMNS, SweepRow, SweepSpec, measure_throughput, read_csv,
                                         run_sweep, write_csv)

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "golden_sweep.json").read_text())
KEEP = ("e", "u", "R", "f", "frames", "success_rate", "mean_iterations", "residual_error_rate")


def test_csv_v1_schema_and_roundtrip():
    rows = [SweepRow(0.03, 2, 0.5, 2.5721241906809027, 24, 1.0, 2.0, 123.5, 0.25, 0.0),
            SweepRow(0.2, 1, 0.5, 0.69, 0, 0.0, 0.0, 0.0, 0.0, 0.0)]
    sink = io.StringIO()
    write_csv(rows, sink)
    text = sink.getvalue().splitlines()
    assert text[:5] == GOLD["csv_header"]
    assert tuple(text[4].split(",")) == CSV_COLUMNS
    assert read_csv(io.StringIO(sink.getvalue())) == rows


def test_spec_validation():
    with pytest.raises(ValueError, match="frames per point"):
        SweepSpec((0.03,), (1,), {0.5: object()}, 0)


@pytest.mark.gpu
def test_run_sweep_matches_reference(cfg1_ensemble):
    spec = SweepSpec(e_values=(0.03, 0.09, 0.2), u_values=(1, 2), ensembles={0.5: cfg1_ensemble}, frames=24,
                     warmup=2, seed=3)
    sink = io.StringIO()
    rows = run_sweep(spec, sink)
    assert len(rows) == len(GOLD["rows"])
    for r, g in zip(rows, GOLD["rows"]):
        for k in KEEP:
            assert getattr(r, k) == g[k], (k, r, g)
    assert read_csv(io.StringIO(sink.getvalue())) == rows


@pytest.mark.gpu
@pytest.mark.parametrize("name,kw", [("prior", dict(prior_e=0.05)), ("calibrate", dict(calibrate=True))])
def test_measure_throughput_modes_match_reference(cfg1_ensemble, name, kw):
    p = measure_throughput(cfg1_ensemble, 2, 0.07, frames=20, seed=4, warmup=1, point_path=(5,), **kw)
    g = GOLD["points"][name]
    for k in ("mean_iterations", "success_rate", "residual_error_rate", "frames"):
        assert getattr(p, k) == g[k], k
    assert abs(p.iterations_std - g["iterations_std"]) < 1e-12


@pytest.mark.gpu
def test_cli_backend_hook_runs_the_reference_sweep(cfg1_ensemble):
    """The names cli_backend.install puts into mmrecon.cli give the
    reference's rows (the same golden as run_sweep above)."""
    import types

    from paper_2001_07979_b200 import cli_backend

    mod = types.SimpleNamespace(measure_throughput=None, run_sweep=None)
    cli_backend.install(mod)
    spec = SweepSpec(e_values=(0.03, 0.09, 0.2), u_values=(1, 2), ensembles={0.5: cfg1_ensemble}, frames=24,
                     warmup=2, seed=3)
    rows = mod.run_sweep(spec, io.StringIO())
    for r, g in zip(rows, GOLD["rows"]):
        for k in KEEP:
            assert getattr(r, k) == g[k], (k, r, g)
    p = mod.measure_throughput(cfg1_ensemble, 2, 0.07, 20, seed=4, warmup=1, point_path=(5,), prior_e=0.05)
    g = GOLD["points"]["prior"]
    for k in ("mean_iterations", "success_rate", "residual_error_rate", "frames"):
        assert getattr(p, k) == g[k], k
