"""Golden vectors for the MBP decode path, produced by the REFERENCE itself.

Runs only in the build container (imports /root/reference/pkg/src); the npz
files it writes under tests/golden/ are committed and are what the oracle
(tests/test_oracle.py) and the CUDA path (tests/test_gpu_parity.py) are pinned
against on the GPU box.  Frames come from the reference's own
``bench._frame_inputs`` (bench.py:123-130) or the test helpers of
test_decoder.py:38-43 / test_equivalence.py:51-55; outputs from
``decoder.decode`` (decoder.py:207-274) with ``track_decisions=True``;
per-iteration posteriors from ``ws.posterior`` after decoding with
``max_iterations=t`` (deterministic, decoder.py:237-266).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden.py [cfg1 mid u1 cfg2 cfg3]
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import numba  # noqa: E402
from mmrecon.bench import _frame_inputs  # noqa: E402  (reference)
from mmrecon.bits import BitBlock  # noqa: E402
from mmrecon.channel import ChannelModel, bsc_corrupt, generate_key  # noqa: E402
from mmrecon.decoder import DecoderConfig, DecoderWorkspace, decode  # noqa: E402
from mmrecon.matrix import DegreeProfile, MatrixEnsemble, ParityCheckMatrix, build_ensemble  # noqa: E402

from paper_2001_07979_b200.matrix import load_ensemble  # noqa: E402

ENS = ROOT / "paper_2001_07979_b200" / "ensembles"


def ref_ensemble(cache_name):
    """Our cached ensemble re-wrapped as the reference's classes (hash-checked)."""
    ours = load_ensemble(ENS / cache_name)
    mats = []
    for h in ours.matrices:
        rows = [np.asarray(h.row_adj(j)) for j in range(h.m)]
        mats.append(ParityCheckMatrix.from_check_adjacency(h.n, h.m, rows))
    ens = MatrixEnsemble(tuple(mats))
    assert ens.content_hashes() == ours.content_hashes()
    return ens


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def meta():
    return {"numpy": np.__version__, "numba": numba.__version__,
            "generator": "tests/golden/make_golden.py (reference mmrecon 0.1.0)"}


def run_frames(ens, u, e, frames, cfg, seed=0, path=(), posterior_frames=0, keep_bits=True):
    """Decode reference frames; returns dict of stacked arrays."""
    sub = ens.prefix(u)
    out = {k: [] for k in ("key", "noisy", "syn", "converged", "iterations", "mismatches",
                           "corrected", "hist_rows", "history")}
    posts = []
    for i in range(frames):
        key, noisy, syns = _frame_inputs(ens, u, e, seed, tuple(path) + (i,))
        ws = DecoderWorkspace(sub, cfg)
        res = decode(sub, noisy, syns, e, cfg, workspace=ws, track_decisions=True)
        out["key"].append(key.data.copy())
        out["noisy"].append(noisy.data.copy())
        out["syn"].append(np.concatenate([z.data for z in syns]))
        out["converged"].append(res.converged)
        out["iterations"].append(res.iterations_used)
        out["mismatches"].append(res.residual_syndrome_mismatches)
        out["corrected"].append(res.corrected.data.copy())
        out["hist_rows"].append(res.decision_history.shape[0])
        out["history"].append(np.packbits(res.decision_history, axis=1, bitorder="little"))
        if i < posterior_frames:
            per_it = np.zeros((cfg.max_iterations + 1, sub.n))
            per_it[0] = ws.priors
            for t in range(1, res.iterations_used + 1):
                ws_t = DecoderWorkspace(sub, cfg)
                c = DecoderConfig(max_iterations=t, llr_clamp=cfg.llr_clamp, damping=cfg.damping,
                                  combining_mode=cfg.combining_mode)
                decode(sub, noisy, syns, e, c, workspace=ws_t)
                per_it[t] = ws_t.posterior
            posts.append(per_it[: res.iterations_used + 1])
    rows = max(out["hist_rows"])
    hist = np.zeros((frames, rows, (sub.n + 7) // 8), dtype=np.uint8)
    for i, h in enumerate(out["history"]):
        hist[i, : h.shape[0]] = h
    d = {
        "converged": np.array(out["converged"]), "iterations": np.array(out["iterations"], np.int32),
        "mismatches": np.array(out["mismatches"], np.int64), "corrected": np.stack(out["corrected"]),
        "hist_rows": np.array(out["hist_rows"], np.int32), "history": hist,
    }
    if keep_bits:
        d.update(key=np.stack(out["key"]), noisy=np.stack(out["noisy"]), syn=np.stack(out["syn"]))
    else:
        d.update(key_sha=np.array([sha(k) for k in out["key"]]),
                 corrected_sha=np.array([sha(c) for c in out["corrected"]]))
        del d["corrected"], d["history"]
    if posterior_frames:
        maxit = max(p.shape[0] for p in posts)
        P = np.full((posterior_frames, maxit, sub.n), np.nan)
        for i, p in enumerate(posts):
            P[i, : p.shape[0]] = p
        d["posterior"] = P
    return d


def save(name, arrays):
    arrays = dict(arrays)
    for k, v in meta().items():
        arrays[f"meta_{k}"] = np.array(v)
    np.savez_compressed(OUT / name, **arrays)
    print(f"{name}: {(OUT / name).stat().st_size} bytes", flush=True)


def golden_cfg1():
    ens = ref_ensemble("cfg1_n4096_m2048_u2_s1.npz")
    arrays = {}
    cfg = DecoderConfig()
    for e, frames, pf in ((0.03, 64, 4), (0.07, 32, 2), (0.09, 32, 2), (0.11, 16, 0)):
        tag = f"e{int(round(e * 1000)):03d}"
        d = run_frames(ens, 2, e, frames, cfg, posterior_frames=pf)
        for k, v in d.items():
            arrays[f"{tag}_{k}"] = v
        print(f"cfg1 e={e}: conv {d['converged'].mean():.3f} iters {d['iterations'].mean():.2f}")
    save("golden_cfg1.npz", arrays)


def golden_mid():
    """mid ensemble (tests/conftest.py:17-20) under every DecoderConfig variant."""
    ens = ref_ensemble("mid_n512_m256_u3_s91.npz")
    variants = {
        "default": DecoderConfig(),
        "damp25": DecoderConfig(damping=0.25),
        "isolated": DecoderConfig(combining_mode="isolated-per-matrix"),
        "isodamp": DecoderConfig(combining_mode="isolated-per-matrix", damping=0.5, max_iterations=30),
        "clamp18": DecoderConfig(max_iterations=25, llr_clamp=18.0),
        "clamp3": DecoderConfig(max_iterations=20, llr_clamp=3.0),
    }
    arrays = {}
    for vname, cfg in variants.items():
        for e in (0.05, 0.08, 0.11, 0.3):
            tag = f"{vname}_e{int(round(e * 1000)):03d}"
            for u in (1, 3):
                d = run_frames(ens, u, e, 12, cfg, seed=7, path=(u,), posterior_frames=0)
                if e != 0.08:
                    for k, v in d.items():
                        arrays[f"{tag}_u{u}_{k}"] = v
                    continue
                # final workspace state for frame 0 (one error rate keeps the file small)
                key, noisy, syns = _frame_inputs(ens, u, e, 7, (u, 0))
                ws = DecoderWorkspace(ens.prefix(u), cfg)
                decode(ens.prefix(u), noisy, syns, e, cfg, workspace=ws)
                d["ws_posterior"] = ws.posterior.copy()
                d["ws_v2c"] = ws.v2c.copy()
                d["ws_c2v"] = ws.c2v.copy()
                for k, v in d.items():
                    arrays[f"{tag}_u{u}_{k}"] = v
    arrays["variants"] = np.array(list(variants))
    arrays["variant_params"] = np.array([[c.max_iterations, c.llr_clamp, c.damping,
                                          c.combining_mode == "joint-graph"] for c in variants.values()])
    save("golden_mid.npz", arrays)


def golden_u1():
    """test_equivalence.py:38-60 geometry: u=1, n=256, message-exact final state."""
    ens = build_ensemble(256, 128, DegreeProfile.regular(3), u=1, base_seed=3)
    h = ens.matrices[0]
    cfg = DecoderConfig(max_iterations=30)
    arrays = {"chk_ptr": h.chk_ptr.copy(), "chk_var": h.chk_var.copy()}
    for seed, e in ((0, 0.06), (1, 0.09), (2, 0.14)):
        key = generate_key(256, seed=seed)
        noisy, _ = bsc_corrupt(key, ChannelModel(e, seed=seed + 50_000))
        z = BitBlock.from_bits((h.to_dense().astype(np.int64) @ key.to_bits().astype(np.int64)) % 2)
        ws = DecoderWorkspace(ens, cfg)
        res = decode(ens, noisy, [z], e, cfg, workspace=ws, track_decisions=True)
        t = f"s{seed}"
        arrays.update({f"{t}_key": key.data.copy(), f"{t}_noisy": noisy.data.copy(),
                       f"{t}_syn": z.data.copy(), f"{t}_e": np.array(e),
                       f"{t}_converged": np.array(res.converged),
                       f"{t}_iterations": np.array(res.iterations_used),
                       f"{t}_history": res.decision_history.copy(),
                       f"{t}_v2c": ws.v2c.copy(), f"{t}_c2v": ws.c2v.copy(),
                       f"{t}_posterior": ws.posterior.copy()})
    save("golden_u1.npz", arrays)


def golden_big(name, cache, u, points, frames):
    ens = ref_ensemble(cache)
    arrays = {}
    for e in points:
        tag = f"e{int(round(e * 1000)):03d}"
        d = run_frames(ens, u, e, frames, DecoderConfig(), keep_bits=False)
        for k, v in d.items():
            arrays[f"{tag}_{k}"] = v
        print(f"{name} e={e}: conv {d['converged'].mean():.3f} iters {d['iterations'].mean():.2f}",
              flush=True)
    save(f"golden_{name}.npz", arrays)


if __name__ == "__main__":
    todo = sys.argv[1:] or ["cfg1", "mid", "u1", "cfg2", "cfg3"]
    for t in todo:
        if t == "cfg1":
            golden_cfg1()
        elif t == "mid":
            golden_mid()
        elif t == "u1":
            golden_u1()
        elif t == "cfg2":
            golden_big("cfg2", "cfg2_n65536_m32768_u2_s1.npz", 2, (0.02, 0.03, 0.05), 64)
        elif t == "cfg3":
            golden_big("cfg3", "cfg3_n65536_m14650_u3_s11.npz", 3, (0.03,), 32)
