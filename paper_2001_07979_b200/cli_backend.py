"""``--backend b200`` for the reference's command line.

The reference's ``simulate`` and ``bench`` commands (pkg/src/mmrecon/cli.py:
185-245) call two module-level names, ``measure_throughput`` (cli.py:199)
and ``run_sweep`` (cli.py:236, 241).  This package provides both with the
same signatures and semantics (``sweep.py``: the reference's frame streams,
success rates and iteration counts, CSV v1), decoding on the GPU.
``install`` rebinds those two names in ``mmrecon.cli``; ``main`` is the
reference's CLI with one extra flag:

    python -m paper_2001_07979_b200.cli_backend --backend b200 simulate --matrix-dir M --u 2 --e 0.03 --frames 4096
    python -m paper_2001_07979_b200.cli_backend --backend b200 bench --matrix-dir M --e-values 0.02:0.05:0.01 --out s.csv

``--backend cpu`` (the default) runs the reference unchanged.  Everything
else -- flags, config files, matrix directories, printed lines -- is the
reference's own.  The reference package must be importable (it is not
vendored here); INTEGRATION.md §5 shows the same two-line hook added to
mmrecon itself.
"""

from __future__ import annotations

import sys

BACKENDS = ("cpu", "b200")


def install(cli_module=None, device: int = 0):
    """Point ``cli_module`` (default: ``mmrecon.cli``) at the GPU harness.
    Returns the previous bindings so callers can restore them."""
    from . import sweep

    if cli_module is None:
        import mmrecon.cli as cli_module   # the reference package
    previous = {name: getattr(cli_module, name) for name in ("measure_throughput", "run_sweep")}

    def measure_throughput(ensemble, u, e, frames, decoder=None, workers=1, seed=0, warmup=5, point_path=(),
                           calibrate=False, prior_e=None):
        return sweep.measure_throughput(ensemble, u, e, frames, decoder=decoder, workers=workers, seed=seed,
                                        warmup=warmup, point_path=point_path, calibrate=calibrate,
                                        prior_e=prior_e, device=device)

    def run_sweep(spec, csv_sink=None):
        return sweep.run_sweep(spec, csv_sink, device=device)

    measure_throughput.__doc__ = sweep.measure_throughput.__doc__
    run_sweep.__doc__ = sweep.run_sweep.__doc__
    cli_module.measure_throughput = measure_throughput
    cli_module.run_sweep = run_sweep
    return previous


def split_backend(argv):
    """(backend, remaining argv): ``--backend X`` / ``--backend=X`` anywhere."""
    argv = list(argv)
    backend = "cpu"
    out = []
    k = 0
    while k < len(argv):
        a = argv[k]
        if a == "--backend":
            if k + 1 >= len(argv):
                raise SystemExit("--backend needs a value: " + "|".join(BACKENDS))
            backend = argv[k + 1]
            k += 2
            continue
        if a.startswith("--backend="):
            backend = a.split("=", 1)[1]
        else:
            out.append(a)
        k += 1
    if backend not in BACKENDS:
        raise SystemExit(f"unknown backend {backend!r}; choose from {', '.join(BACKENDS)}")
    return backend, out


def main(argv=None) -> int:
    backend, rest = split_backend(sys.argv[1:] if argv is None else argv)
    import mmrecon.cli as cli   # the reference package

    if backend == "b200":
        install(cli)
    return cli.main(rest)


if __name__ == "__main__":
    sys.exit(main())
