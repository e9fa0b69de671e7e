"""Compaction on vs off on one batch: per-frame differences (debug aid)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2001_07979_b200 import BatchDecoder, DecoderConfig  # noqa: E402
from paper_2001_07979_b200 import _native as N  # noqa: E402
from paper_2001_07979_b200.channel import make_frames  # noqa: E402
from paper_2001_07979_b200.matrix import load_ensemble  # noqa: E402

ens = load_ensemble(ROOT / "paper_2001_07979_b200/ensembles/cfg1_n4096_m2048_u2_s1.npz")
B = int(sys.argv[1]) if len(sys.argv) > 1 else 96
fb = make_frames(ens.n, 0.09, B, seed=11)
d0 = BatchDecoder(ens, B)
syn = d0.syndromes(fb.keys)
on = BatchDecoder(ens, B)
off = BatchDecoder(ens, B, flags=N.MBP_NO_COMPACTION)
a = on.decode(fb.noisy, syn, 0.09)
print("on stats", on.last_stats())
b = off.decode(fb.noisy, syn, 0.09)
print("off stats", off.last_stats())
print("iters off", b.iterations.tolist())
print("iters on ", a.iterations.tolist())
bad = np.flatnonzero((a.iterations != b.iterations) | np.any(a.corrected != b.corrected, axis=1))
print("differing frames", bad.tolist())
for k in bad[:8]:
    print(k, "on", a.converged[k], a.iterations[k], a.mismatches[k], "off", b.converged[k], b.iterations[k], b.mismatches[k],
          "bitdiff", int(np.unpackbits(a.corrected[k] ^ b.corrected[k]).sum()),
          "on==key", bool(np.array_equal(a.corrected[k], fb.keys[k])))
