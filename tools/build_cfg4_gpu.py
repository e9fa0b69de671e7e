"""Build BASELINE configs[3]'s ensemble -- the reference's
build_ensemble(2^20, 2^19, regular(3), u=2, base_seed=1) -- with the device
PEG (mbp_peg_build_device, both members in parallel host threads) and save it
in the package's cache format.  Run on a GPU box:
    MBP_PEG_DEBUG=2 python tools/build_cfg4_gpu.py gpurun_out/cfg4_n1048576_m524288_u2_s1.npz"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2001_07979_b200.matrix import build_ensemble, load_ensemble, save_ensemble  # noqa: E402

out = Path(sys.argv[1])
n, m = 1 << 20, 1 << 19
t0 = time.perf_counter()
ens = build_ensemble(n, m, 3, u=2, base_seed=1, workers=2, device=0)
dt = time.perf_counter() - t0
save_ensemble(ens, out, seeds=[1, 2], note=f"mbp_peg_build_device (exact restatement of the reference's peg_build), "
                                           f"build_ensemble(n={n}, m={m}, regular(3), u=2, base_seed=1), {dt:.0f} s")
back = load_ensemble(out)
assert back.content_hashes() == ens.content_hashes()
print(f"cfg4 built in {dt:.0f} s: {ens.content_hashes()} -> {out} ({out.stat().st_size} bytes)", flush=True)
