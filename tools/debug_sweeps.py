"""Compare device state after t sweeps with the oracle (debug aid)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
from paper_2001_07979_b200 import BatchDecoder, DecoderConfig  # noqa: E402
from paper_2001_07979_b200 import _native as N  # noqa: E402
from paper_2001_07979_b200.matrix import load_ensemble, stacked_layout  # noqa: E402

g = dict(np.load(ROOT / "tests/golden/golden_cfg1.npz"))
ens = load_ensemble(ROOT / "paper_2001_07979_b200/ensembles/cfg1_n4096_m2048_u2_s1.npz")
lay = stacked_layout(ens)
noisy, syn = g["e070_noisy"][:4], g["e070_syn"][:4]
nb = np.unpackbits(noisy[0], count=ens.n, bitorder="little")
mb = (ens.m + 7) // 8
sb = np.concatenate([np.unpackbits(syn[0, l * mb:(l + 1) * mb], count=ens.m, bitorder="little") for l in range(2)])
for prec in ("fp32", "fp64"):
    for t in (1, 2, 3):
        dec = BatchDecoder(ens, 4, DecoderConfig(max_iterations=t, precision=prec), flags=N.MBP_KEEP_STATE)
        res = dec.decode(noisy, syn, 0.07)
        r = oracle.decode(lay, nb, sb, 0.07, max_iterations=t)
        post = dec.posterior(0)
        c2v = dec.c2v(0)
        print(prec, t, "iters", res.iterations[0], r["iterations"], "post err", np.max(np.abs(post - r["posterior"])),
              "c2v err", np.max(np.abs(c2v - r["c2v"])), "c2v[:6]", np.round(c2v[:6], 4), np.round(r["c2v"][:6], 4))
