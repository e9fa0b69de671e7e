"""Time the device PEG against the reference's cached matrices.
    python tools/peg_gpu_time.py n m seed [seed ...]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2001_07979_b200.matrix import load_ensemble, peg_construct  # noqa: E402

n, m = int(sys.argv[1]), int(sys.argv[2])
ref = {}
for p in (ROOT / "paper_2001_07979_b200" / "ensembles").glob(f"*_n{n}_m{m}_*.npz"):
    e = load_ensemble(p)
    base = int(p.stem.split("_s")[-1])
    for l, h in enumerate(e.matrices):
        ref[base + l] = h.content_hash()
for s in map(int, sys.argv[3:]):
    t0 = time.perf_counter()
    h = peg_construct(n, m, 3, seed=s, device=0)
    dt = time.perf_counter() - t0
    print(f"n={n} m={m} seed={s}: {dt:.1f}s hash={h.content_hash()[:16]} ref={ref.get(s, '-')[:16]} "
          f"match={h.content_hash() == ref.get(s)}", flush=True)
