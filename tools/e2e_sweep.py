"""Host-path (mbp_decode_batch) timing vs sub-batch count, and decode-kernel
time vs batch size, cfg2 e=0.03.   python tools/e2e_sweep.py"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2001_07979_b200 import BatchDecoder  # noqa: E402
from paper_2001_07979_b200.channel import make_frames  # noqa: E402
from paper_2001_07979_b200.matrix import load_ensemble  # noqa: E402

ens = load_ensemble(ROOT / "paper_2001_07979_b200/ensembles/cfg2_n65536_m32768_u2_s1.npz")
B = 1024
fb = make_frames(ens.n, 0.03, B, seed=0)
dec = BatchDecoder(ens, B)
dev = torch.device("cuda:0")
syn_d = dec.syndromes(torch.from_numpy(fb.keys).to(dev))
noisy_d = torch.from_numpy(fb.noisy).to(dev)
pin_noisy = torch.from_numpy(fb.noisy).pin_memory().numpy()
pin_syn = syn_d.cpu().pin_memory().numpy()
from paper_2001_07979_b200.decoder import BatchResult  # noqa: E402

pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
out = BatchResult(pin(np.empty_like(fb.noisy)), pin(np.empty(B, np.uint8)), pin(np.empty(B, np.int32)),
                  pin(np.empty(B, np.int32)), ens.n)
for sub in ("1", "2", "3", "4", "6", "8"):
    os.environ["MBP_HOST_SUBBATCHES"] = sub
    ts = []
    for k in range(6):
        dec.decode(pin_noisy, pin_syn, 0.03, out=out)
        if k >= 2:
            ts.append(dec.last_timing(e2e=True)[1])
    print(f"subbatches {sub}: e2e {np.mean(ts):.3f} ms  ({B * ens.n / np.mean(ts) / 1e6:.0f} Mbps)")
for b in (128, 256, 512, 1024):
    ts = []
    for k in range(5):
        dec.decode_device(noisy_d[:b], syn_d[:b], torch.tensor([0.03], dtype=torch.float64, device=dev))
        torch.cuda.synchronize()
        if k >= 1:
            ts.append(dec.last_timing()[0])
    print(f"batch {b}: kernel {np.mean(ts):.3f} ms  ({b * ens.n / np.mean(ts) / 1e6:.0f} Mbps)")
