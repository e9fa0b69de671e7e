"""GPU backend of the reference's benchmark harness:
error-rate x matrix-count x code-rate sweeps with the CSV v1 schema kept
byte-compatible (pkg/src/mmrecon/bench.py:49-60, 223-257).

Same names and semantics as ``mmrecon.bench``: ``SweepSpec``, ``SweepRow``,
``ThroughputPoint``, ``measure_throughput``, ``run_sweep``, ``write_csv``,
``read_csv``, ``CSV_COLUMNS``.  Frames are the reference's counter-based
streams (``_frame_inputs``, bench.py:123-130: frame i of a point uses path
point_path + (i,), warmup frames path + (99, i)), so success rates and
iteration counts equal the reference's for the same spec; only the timing
fields differ.  Decoding runs as batches on the GPU (``BatchDecoder``) instead
of a thread pool of per-frame workspaces; ``workers`` sets the number of host
threads that generate frames (the reference's wall clock, and ours, includes
frame generation, bench.py:165-189).

    python -m paper_2001_07979_b200.sweep --ensemble cfg1 --e 0.03,0.05 --u 1,2 --frames 200
"""

from __future__ import annotations

import csv
import logging
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import IO, Mapping

import numpy as np

from .channel import efficiency, make_frames
from .decoder import BatchDecoder, DecoderConfig, _cfg_of

__all__ = ["SweepSpec", "SweepRow", "ThroughputPoint", "run_sweep", "measure_throughput", "write_csv",
           "read_csv", "CSV_COLUMNS"]

log = logging.getLogger("paper_2001_07979_b200.sweep")

# bench.py:49-60 (format v1)
CSV_COLUMNS = (
    "e", "u", "R", "f", "frames", "success_rate", "mean_iterations",
    "throughput_mbps", "mean_time_ms", "residual_error_rate",
)

CSV_DOC_LINES = (
    "# mmrecon bench sweep, format v1",
    "# throughput_mbps counts successfully reconciled sifted bits only"
    " (converged frames with zero residual errors)",
    "# residual_error_rate = converged frames with residual bit errors / converged frames",
    "# frames=0 marks a grid point skipped as infeasible (f <= 1 at the requested e)",
)


@dataclass(frozen=True)
class SweepSpec:
    """Grid definition (bench.py:63-92); code rates come in via ensembles."""

    e_values: tuple[float, ...]
    u_values: tuple[int, ...]
    ensembles: Mapping[float, object]  # nominal R -> MatrixEnsemble
    frames: int
    decoder: DecoderConfig = field(default_factory=DecoderConfig)
    workers: int = 1
    seed: int = 0
    warmup: int = 5
    k: int = 16

    def __post_init__(self):
        if self.frames < 1:
            raise ValueError(f"frames per point must be >= 1, got {self.frames}")
        if not self.e_values:
            raise ValueError("no error rates given")
        if not self.u_values or min(self.u_values) < 1:
            raise ValueError("u values must be >= 1")
        if not self.ensembles:
            raise ValueError("no ensembles given")
        for r, ens in self.ensembles.items():
            if max(self.u_values) > ens.u:
                raise ValueError(f"ensemble for R={r} has u={ens.u}, sweep needs {max(self.u_values)}")


@dataclass(frozen=True)
class SweepRow:
    e: float
    u: int
    R: float
    f: float
    frames: int
    success_rate: float
    mean_iterations: float
    throughput_mbps: float
    mean_time_ms: float
    residual_error_rate: float


@dataclass(frozen=True)
class ThroughputPoint:
    mbps: float
    mean_time_ms: float
    mean_iteration_time_ms: float
    mean_iterations: float
    iterations_std: float
    success_rate: float
    residual_error_rate: float
    frames: int
    wall_time_s: float


def _gen(n, e, frames, seed, path, workers, chunk=256):
    """make_frames over [0, frames) split into chunks on `workers` threads."""
    if workers <= 1 or frames <= chunk:
        fb = make_frames(n, e, frames, seed=seed, path=path)
        return fb.keys, fb.noisy
    starts = list(range(0, frames, chunk))
    with ThreadPoolExecutor(max_workers=workers) as pool:
        parts = list(pool.map(lambda s: make_frames(n, e, min(chunk, frames - s), seed=seed, path=path, start=s),
                              starts))
    return np.concatenate([p.keys for p in parts]), np.concatenate([p.noisy for p in parts])


_DECODERS: dict = {}


def _decoder_for(sub, cfg, batch, device):
    """One device workspace per (matrix set, config, batch, device): grid
    points of a sweep reuse it (``prefix(u)`` builds a new ensemble object
    per call, so the key is the matrices' content hashes)."""
    key = (tuple(sub.content_hashes()), cfg, batch, device)
    dec = _DECODERS.get(key)
    if dec is None:
        if len(_DECODERS) >= 8:   # bound the device memory held by the cache
            _DECODERS.pop(next(iter(_DECODERS)))
        dec = _DECODERS[key] = BatchDecoder(sub, batch, cfg, device=device)
    return dec


def measure_throughput(ensemble, u: int, e: float, frames: int, decoder=None, workers: int = 1, seed: int = 0,
                       warmup: int = 5, point_path: tuple = (), calibrate: bool = False,
                       prior_e: float | None = None, batch: int = 4096, device: int = 0) -> ThroughputPoint:
    """One grid point (bench.py:133-204): warmup frames, then timed frames.

    ``calibrate=True`` replaces the decoder by a no-op (harness overhead);
    ``prior_e`` lets the decoder assume a misestimated crossover probability
    while the channel keeps the true ``e``."""
    cfg = _cfg_of(decoder)
    assumed_e = e if prior_e is None else prior_e
    sub = ensemble.prefix(u)
    n = ensemble.n
    dec = None if calibrate else _decoder_for(sub, cfg, min(batch, max(frames, warmup, 1)), device)

    def run(path, count):
        """Frames 0..count-1 of `path`: generate, syndromes, decode in
        batches; returns (converged, iterations, residual_zero, decode_s)."""
        keys, noisy = _gen(n, e, count, seed, path, workers)
        if calibrate:   # no-op decoder: "corrected" = the noisy key (bench.py:166-167)
            return (np.ones(count, bool), np.zeros(count, np.int64), np.all(noisy == keys, axis=1), 0.0)
        conv = np.empty(count, bool)
        its = np.empty(count, np.int64)
        clean = np.empty(count, bool)
        dt = 0.0
        for lo in range(0, count, dec.max_frames):
            hi = min(count, lo + dec.max_frames)
            syn = dec.syndromes(keys[lo:hi])
            t0 = time.perf_counter()
            r = dec.decode(noisy[lo:hi], syn, assumed_e)
            dt += time.perf_counter() - t0
            conv[lo:hi] = r.converged
            its[lo:hi] = r.iterations
            clean[lo:hi] = np.all(r.corrected == keys[lo:hi], axis=1)
        return conv, its, clean, dt

    if warmup:
        run(tuple(point_path) + (99,), warmup)
    wall0 = time.perf_counter()
    conv, its, clean, decode_time = run(tuple(point_path), frames)
    wall = time.perf_counter() - wall0

    good = conv & clean
    n_conv = int(conv.sum())
    total_iters = int(its.sum())
    iters = its.astype(np.float64)
    return ThroughputPoint(
        mbps=int(good.sum()) * n / wall / 1e6 if wall > 0 else 0.0,
        mean_time_ms=1e3 * decode_time / frames,
        mean_iteration_time_ms=1e3 * decode_time / total_iters if total_iters else 0.0,
        mean_iterations=float(iters.mean()),
        iterations_std=float(iters.std()),
        success_rate=n_conv / frames,
        residual_error_rate=(n_conv - int(good.sum())) / n_conv if n_conv else 0.0,
        frames=frames,
        wall_time_s=wall,
    )


def run_sweep(spec: SweepSpec, csv_sink: IO[str] | None = None, device: int = 0) -> list[SweepRow]:
    """The full grid (bench.py:207-242); emits CSV v1 if a sink is given."""
    rows: list[SweepRow] = []
    for r_nominal in sorted(spec.ensembles):
        ensemble = spec.ensembles[r_nominal]
        for u in spec.u_values:
            for e in spec.e_values:
                f = efficiency(ensemble.m, ensemble.n, e)
                if f <= 1.0:
                    log.warning("skipping infeasible point R=%s u=%d e=%.4f (f=%.4f <= 1)", r_nominal, u, e, f)
                    rows.append(SweepRow(e, u, r_nominal, f, 0, 0.0, 0.0, 0.0, 0.0, 0.0))
                    continue
                point_path = (int(round(r_nominal * 1e6)), int(round(e * 1e6)))
                p = measure_throughput(ensemble, u, e, frames=spec.frames, decoder=spec.decoder,
                                       workers=spec.workers, seed=spec.seed, warmup=spec.warmup,
                                       point_path=point_path, device=device)
                rows.append(SweepRow(e=e, u=u, R=r_nominal, f=f, frames=p.frames, success_rate=p.success_rate,
                                     mean_iterations=p.mean_iterations, throughput_mbps=p.mbps,
                                     mean_time_ms=p.mean_time_ms, residual_error_rate=p.residual_error_rate))
    if csv_sink is not None:
        write_csv(rows, csv_sink)
    return rows


def write_csv(rows: list[SweepRow], sink: IO[str]) -> None:
    """bench.py:245-257."""
    for line in CSV_DOC_LINES:
        sink.write(line + "\n")
    writer = csv.writer(sink)
    writer.writerow(CSV_COLUMNS)
    for row in rows:
        writer.writerow([
            repr(row.e), row.u, repr(row.R), repr(row.f), row.frames,
            repr(row.success_rate), repr(row.mean_iterations),
            repr(row.throughput_mbps), repr(row.mean_time_ms),
            repr(row.residual_error_rate),
        ])


def read_csv(source: IO[str]) -> list[SweepRow]:
    """bench.py:260-277."""
    lines = [ln for ln in source if not ln.startswith("#")]
    reader = csv.reader(lines)
    header = next(reader)
    if tuple(header) != CSV_COLUMNS:
        raise ValueError(f"unexpected CSV columns {header}")
    out = []
    for rec in reader:
        if not rec:
            continue
        out.append(SweepRow(e=float(rec[0]), u=int(rec[1]), R=float(rec[2]), f=float(rec[3]), frames=int(rec[4]),
                            success_rate=float(rec[5]), mean_iterations=float(rec[6]),
                            throughput_mbps=float(rec[7]), mean_time_ms=float(rec[8]),
                            residual_error_rate=float(rec[9])))
    return out


def _parse_floats(text):
    if ":" in text:
        a, b, s = (float(x) for x in text.split(":"))
        k = int(round((b - a) / s))
        return tuple(round(a + i * s, 10) for i in range(k + 1))
    return tuple(float(x) for x in text.split(","))


def main(argv=None) -> int:
    import argparse
    import sys
    from pathlib import Path

    from .matrix import load_ensemble

    ap = argparse.ArgumentParser(prog="python -m paper_2001_07979_b200.sweep",
                                 description="GPU sweep: e x u x R grid, CSV v1 (mmrecon bench format)")
    ap.add_argument("--ensemble", action="append", required=True,
                    help="ensemble cache name under ensembles/ (e.g. cfg2) or a .npz path; repeatable")
    ap.add_argument("--e", dest="e_values", default="0.03:0.10:0.01")
    ap.add_argument("--u", dest="u_values", default="1,2")
    ap.add_argument("--frames", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--workers", type=int, default=4)
    ap.add_argument("--out")
    a = ap.parse_args(argv)
    here = Path(__file__).resolve().parent / "ensembles"
    ensembles = {}
    for name in a.ensemble:
        p = Path(name)
        ens = load_ensemble(p if p.suffix == ".npz" else next(here.glob(f"{name}_*.npz")))
        ensembles[round(1.0 - ens.m / ens.n, 6)] = ens
    spec = SweepSpec(e_values=_parse_floats(a.e_values), u_values=tuple(int(x) for x in a.u_values.split(",")),
                     ensembles=ensembles, frames=a.frames, workers=a.workers, seed=a.seed, warmup=a.warmup)
    if a.out:
        with open(a.out, "w", newline="") as fh:
            rows = run_sweep(spec, fh)
        print(f"{len(rows)} rows -> {a.out}")
    else:
        run_sweep(spec, sys.stdout)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
