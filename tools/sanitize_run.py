"""Small decodes for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [--quick]

Runs every kernel family of libmbp_b200.so once on small inputs: syndrome +
transposes, the scatter decode (cfg 1 with and without compaction, random
irregular ensembles with wide rows), the explicit-message decode (fp32, fp64,
damping, isolated), the single-phase kernels; each result is checked against
the oracle so a sanitizer-clean run is also a correct one.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle  # noqa: E402
from paper_2001_07979_b200 import BatchDecoder, DecoderConfig  # noqa: E402
from paper_2001_07979_b200 import _native as N  # noqa: E402
from paper_2001_07979_b200.channel import make_frames  # noqa: E402
from paper_2001_07979_b200.matrix import load_ensemble, stacked_layout  # noqa: E402


def check(ens, fb, dec, e, cfg, label):
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, e)
    lay = stacked_layout(ens)
    og = oracle.OracleGraph(lay)
    u, m = ens.u, ens.m
    mb = (m + 7) // 8
    bad = 0
    for k in range(fb.batch):
        zs = np.concatenate([np.unpackbits(syn[k, l * mb:(l + 1) * mb], count=m, bitorder="little")
                             for l in range(u)])
        r = oracle.decode(og, np.unpackbits(fb.noisy[k], count=ens.n, bitorder="little"), zs, e,
                          max_iterations=cfg.max_iterations, clamp=cfg.llr_clamp, damping=cfg.damping,
                          joint=cfg.combining_mode == "joint-graph")
        bad += (bool(res.converged[k]) != r["converged"]) or (int(res.iterations[k]) != r["iterations"])
    print(f"{label}: {fb.batch} frames, mismatching frames vs oracle: {bad}", flush=True)
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="cfg 1 only (racecheck is slow)")
    a = ap.parse_args()
    from test_gpu_scatter import _random_ensemble

    ens = load_ensemble(ROOT / "paper_2001_07979_b200" / "ensembles" / "cfg1_n4096_m2048_u2_s1.npz")
    bad = 0
    fb = make_frames(ens.n, 0.08, 64, seed=0, path=(3,))
    for flags, label in ((0, "scatter"), (N.MBP_NO_COMPACTION, "scatter/no-compaction"),
                         (N.MBP_EXPLICIT_MESSAGES, "explicit fp32")):
        cfg = DecoderConfig(max_iterations=12)
        bad += check(ens, fb, BatchDecoder(ens, 64, cfg, flags=flags), 0.08, cfg, f"cfg1 e=0.08 {label}")
    if not a.quick:
        for kw, label in ((dict(precision="fp64"), "fp64"), (dict(damping=0.3), "damping"),
                          (dict(combining_mode="isolated-per-matrix"), "isolated")):
            cfg = DecoderConfig(max_iterations=10, **kw)
            bad += check(ens, fb, BatchDecoder(ens, 64, cfg), 0.08, cfg, f"cfg1 e=0.08 {label}")
        for seed in range(3):
            rng = np.random.default_rng(1000 + seed)
            rens = _random_ensemble(rng, int(rng.integers(1, 4)))
            e = float(rng.uniform(0.01, 0.08))
            B = int(rng.integers(33, 100))
            cfg = DecoderConfig(max_iterations=15)
            rfb = make_frames(rens.n, e, B, seed=seed)
            bad += check(rens, rfb, BatchDecoder(rens, B, cfg), e, cfg, f"random irregular #{seed}")
        # single-phase kernels through the reference-shaped API
        from paper_2001_07979_b200 import decoder as D
        from paper_2001_07979_b200.bits import BitBlock

        ws = D.DecoderWorkspace(ens)
        ws.priors[:] = D.init_priors(BitBlock.from_bits(np.unpackbits(fb.noisy[0], count=ens.n,
                                                                      bitorder="little")), 0.05)
        ws.v2c[:] = ws.priors[ws.chk_var]
        syn = dec_syn = BatchDecoder(ens, 1).syndromes(fb.keys[:1])
        mb = (ens.m + 7) // 8
        for l in range(ens.u):
            D.c2v_update(ws, l, BitBlock.from_bits(np.unpackbits(syn[0, l * mb:(l + 1) * mb], count=ens.m,
                                                                 bitorder="little")))
        for l in range(ens.u):
            D.v2c_update(ws, l)
        D.soft_decision(ws)
        del dec_syn
        print("single-phase kernels ran", flush=True)
    print(f"SANITIZE_RUN_DONE bad={bad}", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
