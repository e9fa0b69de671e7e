"""The --backend b200 hook for the reference CLI (paper_2001_07979_b200/
cli_backend.py): argument handling and the rebinding of the two names the
reference's simulate / bench commands call (cli.py:199, 236-241).  Host
only; the GPU harness behind them is tested in test_sweep.py."""

import sys
import types
from pathlib import Path

import pytest

from paper_2001_07979_b200 import cli_backend, sweep


def test_split_backend():
    assert cli_backend.split_backend(["simulate", "--e", "0.03"]) == ("cpu", ["simulate", "--e", "0.03"])
    assert cli_backend.split_backend(["--backend", "b200", "bench", "--out", "x"]) == ("b200", ["bench", "--out", "x"])
    assert cli_backend.split_backend(["simulate", "--backend=b200"]) == ("b200", ["simulate"])
    with pytest.raises(SystemExit):
        cli_backend.split_backend(["--backend", "tpu", "simulate"])
    with pytest.raises(SystemExit):
        cli_backend.split_backend(["simulate", "--backend"])


def test_install_rebinds_harness_names():
    mod = types.SimpleNamespace(measure_throughput=lambda *a, **k: "ref-point", run_sweep=lambda *a, **k: "ref-rows")
    prev = cli_backend.install(mod)
    assert prev["measure_throughput"]() == "ref-point" and prev["run_sweep"]() == "ref-rows"
    assert mod.measure_throughput.__doc__ == sweep.measure_throughput.__doc__
    assert mod.run_sweep.__doc__ == sweep.run_sweep.__doc__


def test_install_into_the_reference_cli():
    ref = Path("/root/reference/pkg/src")
    if not ref.exists():
        pytest.skip("reference package not present (build container only)")
    sys.path.insert(0, str(ref))
    try:
        cli = pytest.importorskip("mmrecon.cli")
        prev = cli_backend.install(cli)
        try:
            assert cli.measure_throughput is not prev["measure_throughput"]
            assert cli.run_sweep is not prev["run_sweep"]
            # the reference's commands resolve the names at call time
            assert "measure_throughput(" in Path(cli.__file__).read_text()
        finally:
            cli.measure_throughput = prev["measure_throughput"]
            cli.run_sweep = prev["run_sweep"]
    finally:
        sys.path.remove(str(ref))
