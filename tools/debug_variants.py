"""Decode every golden_mid variant in order, printing each tag first (finds
the first case a library variant fails on).  MBP_LIB selects the library."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
from conftest import load_golden, _ens
from paper_2001_07979_b200 import BatchDecoder, DecoderConfig
from paper_2001_07979_b200 import _native as N

g = load_golden("golden_mid.npz")
mid = _ens("mid")
for vi, vname in enumerate(g["variants"]):
    max_it, clamp, damping, joint = g["variant_params"][vi]
    cfg = DecoderConfig(int(max_it), float(clamp), float(damping),
                        "joint-graph" if joint else "isolated-per-matrix", sys.argv[1] if len(sys.argv) > 1 else "fp32")
    for u in (1, 3):
        ens = mid.prefix(u)
        for e in ("050", "080", "110", "300"):
            for fl in (0, N.MBP_RECORD_HISTORY):
                tag = f"{vname}_e{e}_u{u}"
                print(tag, "flags", fl, flush=True)
                dec = BatchDecoder(ens, g[f"{tag}_noisy"].shape[0], cfg, flags=fl)
                res = dec.decode(g[f"{tag}_noisy"], g[f"{tag}_syn"], int(e) / 1000)
                print("  ok", np.array_equal(res.iterations, g[f"{tag}_iterations"]), flush=True)
