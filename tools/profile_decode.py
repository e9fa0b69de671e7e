"""Per-phase device timing of the decode kernel (MBP_PROFILE_PHASES stamps).

    python tools/profile_decode.py [--cfg cfg2] [--frames 1024] [--e 0.03] [--once]

--once: a single warm decode (for `ncu -k regex:decode_kernel -c 1`).
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2001_07979_b200 import BatchDecoder, DecoderConfig  # noqa: E402
from paper_2001_07979_b200 import _native as N  # noqa: E402
from paper_2001_07979_b200.channel import make_frames_native as make_frames  # noqa: E402
from paper_2001_07979_b200.matrix import load_ensemble  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg2")
    ap.add_argument("--frames", type=int, default=1024)
    ap.add_argument("--e", type=float, default=0.03)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-compact", action="store_true")
    a = ap.parse_args()
    import torch

    ens = load_ensemble(next((ROOT / "paper_2001_07979_b200" / "ensembles").glob(f"{a.cfg}_*.npz")))
    fb = make_frames(ens.n, a.e, a.frames, seed=0)
    flags = (0 if a.once else N.MBP_PROFILE_PHASES) | (N.MBP_NO_COMPACTION if a.no_compact else 0)
    dec = BatchDecoder(ens, a.frames, DecoderConfig(precision=a.precision), flags=flags)
    dev = torch.device("cuda:0")
    keys = torch.from_numpy(fb.keys).to(dev)
    noisy = torch.from_numpy(fb.noisy).to(dev)
    syn = dec.syndromes(keys)
    e = torch.tensor([a.e], dtype=torch.float64, device=dev)
    out = dec.decode_device(noisy, syn, e)
    torch.cuda.synchronize()
    if a.once:
        return
    res = []
    for _ in range(a.reps):
        dec.decode_device(noisy, syn, e, out=out)
        torch.cuda.synchronize()
        kms, sweeps = dec.last_timing()
        res.append({"kernel_ms": kms, "compaction_sweep": dec.last_stats()[1], **dec.phase_times()})
    it = out[2].cpu().numpy()
    ok = out[1].cpu().numpy().astype(bool) & np.all(out[0].cpu().numpy() == fb.keys, axis=1)
    print(json.dumps({"cfg": a.cfg, "frames": a.frames, "e": a.e, "precision": a.precision,
                      "mean_iterations": float(it.mean()),
                      "iteration_histogram": {int(k): int(v) for k, v in zip(*np.unique(it, return_counts=True))}, "good": int(ok.sum()), "runs": res}, indent=1))


if __name__ == "__main__":
    main()
