"""Decode one golden_mid case: python tools/debug_case.py TAG FLAGS [precision]
(e.g. default_e110_u3 8); prints iterations equality with the golden."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
from conftest import load_golden, _ens
from paper_2001_07979_b200 import BatchDecoder, DecoderConfig

tag, fl = sys.argv[1], int(sys.argv[2])
g = load_golden("golden_mid.npz")
vname, e, u = tag.split("_")
vi = list(g["variants"]).index(vname)
max_it, clamp, damping, joint = g["variant_params"][vi]
import os
max_it = int(os.environ.get("MAXIT", max_it))
cfg = DecoderConfig(int(max_it), float(clamp), float(damping), "joint-graph" if joint else "isolated-per-matrix",
                    sys.argv[3] if len(sys.argv) > 3 else "fp32")
ens = _ens("mid").prefix(int(u[1:]))
dec = BatchDecoder(ens, g[f"{tag}_noisy"].shape[0], cfg, flags=fl)
res = dec.decode(g[f"{tag}_noisy"], g[f"{tag}_syn"], int(e[1:]) / 1000)
print(tag, fl, "maxit", max_it, "iters ok", np.array_equal(res.iterations, g[f"{tag}_iterations"]), "frames", len(res.iterations),
      "iters", np.bincount(res.iterations), "sweeps", dec.last_stats() if hasattr(dec, "last_stats") else None)
