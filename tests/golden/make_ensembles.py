"""Build the PEG ensembles of SURVEY.md §8(d) with the REFERENCE's own
``build_ensemble`` (pkg/src/mmrecon/matrix.py:238-260) and store them in the
package's compact cache format (paper_2001_07979_b200/matrix.py).

Runs only in the build container (it imports /root/reference); the caches it
writes are committed under paper_2001_07979_b200/ensembles/ so the GPU box,
which has no /root/reference, decodes on exactly the reference's matrices.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_ensembles.py cfg1 cfg2 cfg3
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from mmrecon.matrix import DegreeProfile, build_ensemble  # noqa: E402  (reference)

from paper_2001_07979_b200.matrix import load_ensemble, save_ensemble  # noqa: E402

# name -> (n, m, u, base_seed)
SPECS = {
    "cfg1": (4096, 2048, 2, 1),
    "cfg2": (65536, 32768, 2, 1),
    "cfg3": (65536, 14650, 3, 11),
    "cfg4": (1 << 20, 1 << 19, 2, 1),   # BASELINE configs[3]: ~7 h per matrix in the reference
    "mid": (512, 256, 3, 91),      # reference tests/conftest.py:17-20
    "toy": (64, 32, 3, 41),        # reference tests/conftest.py:11-14
    "desk": (16384, 8192, 3, 1001),  # reference test_acceptance.py:53-59
}

if __name__ == "__main__":
    import os

    out = Path(os.environ.get("ENSEMBLE_OUT", ROOT / "paper_2001_07979_b200" / "ensembles"))
    out.mkdir(parents=True, exist_ok=True)
    for name in sys.argv[1:]:
        n, m, u, seed = SPECS[name]
        t0 = time.perf_counter()
        ens = build_ensemble(n, m, DegreeProfile.regular(3), u=u, base_seed=seed, workers=u)
        path = out / f"{name}_n{n}_m{m}_u{u}_s{seed}.npz"
        save_ensemble(ens, path, seeds=[seed + l for l in range(u)],
                      note=f"reference build_ensemble(n={n}, m={m}, regular(3), u={u}, base_seed={seed})")
        back = load_ensemble(path)
        assert back.content_hashes() == ens.content_hashes()
        print(f"{name}: built in {time.perf_counter() - t0:.1f}s -> {path.name} "
              f"({path.stat().st_size} bytes)", flush=True)
