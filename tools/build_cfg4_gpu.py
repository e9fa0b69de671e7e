"""Build BASELINE configs[3]'s ensemble -- the reference's
build_ensemble(2^20, 2^19, regular(3), u=2, base_seed=1) -- with the device
PEG (both members in parallel host threads) and save it in the package's
cache format.  Resumable: with --until V it stops after variable V and writes
a checkpoint (per-variable check lists + tie-break stream states); --resume
continues from one.  Run on a GPU box:

    MBP_PEG_DEBUG=2 python tools/build_cfg4_gpu.py --until 786432 --ckpt gpurun_out/cfg4_ckpt.npz
    MBP_PEG_DEBUG=2 python tools/build_cfg4_gpu.py --resume gpurun_out/cfg4_ckpt.npz \\
        --out gpurun_out/cfg4_n1048576_m524288_u2_s1.npz
"""
import argparse
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2001_07979_b200.matrix import (MatrixEnsemble, load_ensemble, matrix_from_variable_rows,  # noqa: E402
                                          peg_device_stage, save_ensemble)

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--m", type=int, default=1 << 19)
ap.add_argument("--seeds", default="1,2")
ap.add_argument("--until", type=int, default=None, help="stop after this many variables (checkpoint)")
ap.add_argument("--resume", help="checkpoint to continue from")
ap.add_argument("--ckpt", help="checkpoint to write when stopping early")
ap.add_argument("--out", help="ensemble cache to write when complete")
a = ap.parse_args()
n, m = a.n, a.m
seeds = [int(x) for x in a.seeds.split(",")]
if a.resume:
    z = np.load(a.resume)
    v0 = int(z["v"])
    rows = [np.ascontiguousarray(z[f"rows{i}"]) for i in range(len(seeds))]
    states = [int(x) for x in z["states"]]
else:
    v0 = 0
    rows = [np.full((n, 4), -1, dtype=np.int32) for _ in seeds]
    states = [0 for _ in seeds]
v1 = n if a.until is None else min(n, a.until)
t0 = time.perf_counter()
with ThreadPoolExecutor(len(seeds)) as pool:
    states = list(pool.map(lambda i: peg_device_stage(n, m, 3, seeds[i], states[i], v0, v1, rows[i], 0),
                           range(len(seeds))))
dt = time.perf_counter() - t0
print(f"variables [{v0}, {v1}) in {dt:.0f} s", flush=True)
if v1 < n:
    np.savez_compressed(a.ckpt, v=np.array(v1), states=np.array(states, dtype=np.uint64),
                        **{f"rows{i}": r for i, r in enumerate(rows)})
    print(f"checkpoint -> {a.ckpt}", flush=True)
else:
    ens = MatrixEnsemble(tuple(matrix_from_variable_rows(n, m, r) for r in rows))
    save_ensemble(ens, a.out, seeds=seeds,
                  note=f"mbp_peg_build_device (exact restatement of the reference's peg_build), "
                       f"build_ensemble(n={n}, m={m}, regular(3), u={len(seeds)}, base_seed={seeds[0]})")
    back = load_ensemble(a.out)
    assert back.content_hashes() == ens.content_hashes()
    print(f"built: {ens.content_hashes()} -> {a.out} ({Path(a.out).stat().st_size} bytes)", flush=True)
