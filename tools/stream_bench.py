"""Decode-kernel time per 1024 frames for streams of several lengths (one
launch each; waves of 1024 frames), cfg/e from the command line.
    python tools/stream_bench.py [cfg2] [0.03]"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2001_07979_b200 import BatchDecoder  # noqa: E402
from paper_2001_07979_b200.channel import make_frames  # noqa: E402
from paper_2001_07979_b200.matrix import load_ensemble  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
e = float(sys.argv[2]) if len(sys.argv) > 2 else 0.03
ens = load_ensemble(next((ROOT / "paper_2001_07979_b200/ensembles").glob(f"{cfg}_*.npz")))
fb = make_frames(ens.n, e, 1024, seed=0)
dev = torch.device("cuda:0")
dec = BatchDecoder(ens, 1024)
keys = torch.from_numpy(fb.keys).to(dev)
noisy1 = torch.from_numpy(fb.noisy).to(dev)
syn1 = dec.syndromes(keys)
ed = torch.tensor([e], dtype=torch.float64, device=dev)
ref = dec.decode_device(noisy1, syn1, ed)
torch.cuda.synchronize()
ref = [x.cpu().numpy() for x in ref]
for reps in (1, 4, 16):
    noisy = noisy1.repeat(reps, 1)
    syn = syn1.repeat(reps, 1)
    ts = []
    for k in range(4):
        out = dec.decode_device(noisy, syn, ed)
        torch.cuda.synchronize()
        if k:
            ts.append(dec.last_timing()[0])
    o = [x.cpu().numpy() for x in out]
    same = all(np.array_equal(o[i], np.tile(ref[i], (reps,) + (1,) * (ref[i].ndim - 1))) for i in range(4))
    ms = float(np.mean(ts))
    print(f"{cfg} e={e} stream {reps}x1024: kernel {ms:.3f} ms = {ms / reps:.3f} ms/1024 frames "
          f"({reps * 1024 * ens.n / ms / 1e6:.0f} Mbps)  identical_to_single={same}")
