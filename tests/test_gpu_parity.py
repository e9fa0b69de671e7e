"""Parity of the CUDA decode path (through the C ABI) with the oracle and the
reference's golden vectors.  Contract:

* syndromes: bit-exact;
* per frame: ``converged``, ``iterations_used``, ``residual_syndrome_mismatches``
  and the per-sweep decision history equal; corrected bits of converged
  frames equal;
* posterior LLRs after every sweep within |d| <= 1e-4 * max(|ref|, 1) in the
  fp32 production path, <= 1e-9 * max(|ref|, 1) in fp64 parity mode.
"""

import hashlib

import numpy as np
import pytest

import oracle
from paper_2001_07979_b200 import BatchDecoder, DecoderConfig
from paper_2001_07979_b200 import _native as N
from paper_2001_07979_b200.bits import pack_rows, unpack_rows
from paper_2001_07979_b200.channel import make_frames
from paper_2001_07979_b200.matrix import MatrixEnsemble, ParityCheckMatrix, stacked_layout

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "fp64": 1e-9}


def rel_err(got, ref):
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)))


def syn_bits_of(rows, u, m):
    mb = (m + 7) // 8
    return np.concatenate([unpack_rows(rows[:, l * mb:(l + 1) * mb], m) for l in range(u)], axis=1)


# ---------------------------------------------------------------------------
# syndromes (Alice side)
# ---------------------------------------------------------------------------

def test_syndromes_match_golden(golden_cfg1, cfg1_ensemble):
    dec = BatchDecoder(cfg1_ensemble, 64)
    for tag in ("e030", "e070"):
        got = dec.syndromes(golden_cfg1[f"{tag}_key"])
        assert np.array_equal(got, golden_cfg1[f"{tag}_syn"])


def _random_matrix(rng):
    n = int(rng.integers(24, 1025))
    m = int(rng.integers(8, n))
    rows = [[] for _ in range(m)]
    for i in range(n):
        for c in rng.choice(m, size=int(rng.integers(1, min(4, m) + 1)), replace=False):
            rows[int(c)].append(i)
    rows = [r for r in rows if r]
    if not 0 < len(rows) < n:
        return None
    return ParityCheckMatrix.from_check_adjacency(n, len(rows), rows)


def test_syndromes_random_matrices_vs_dense():
    """criterion 2 (test_acceptance.py:111-124) on ragged shapes and batches."""
    rng = np.random.default_rng(404)
    done = 0
    while done < 40:
        h = _random_matrix(rng)
        if h is None:
            continue
        B = int(rng.choice([1, 7, 32, 33, 70]))
        keys = rng.integers(0, 2, size=(B, h.n), dtype=np.uint8)
        dec = BatchDecoder(h, B)
        got = unpack_rows(dec.syndromes(pack_rows(keys)), h.m)
        dense = (keys.astype(np.int64) @ h.to_dense().T.astype(np.int64)) % 2
        assert np.array_equal(got, dense)
        done += 1


def test_syndromes_full_size_vs_oracle_and_linearity(cfg3_ensemble):
    lay = stacked_layout(cfg3_ensemble)
    rng = np.random.default_rng(5)
    B = 40
    keys = rng.integers(0, 2, size=(B, lay.n), dtype=np.uint8)
    dec = BatchDecoder(cfg3_ensemble, B)
    rows = dec.syndromes(pack_rows(keys))
    bits = syn_bits_of(rows, lay.u, lay.m)
    for k in (0, 17, 39):
        assert np.array_equal(bits[k], oracle.syndrome(lay.chk_ptr, lay.chk_var, keys[k]))
    a, b = pack_rows(keys[:20]), pack_rows(keys[20:])
    assert np.array_equal(dec.syndromes(a ^ b), rows[:20] ^ rows[20:])


# ---------------------------------------------------------------------------
# decode against golden frames
# ---------------------------------------------------------------------------

def _decode_rows(ens, noisy, syn, e, cfg, flags=0):
    dec = BatchDecoder(ens, noisy.shape[0], cfg, flags=flags)
    return dec, dec.decode(noisy, syn, e)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("tag", ["e030", "e070", "e090", "e110"])
def test_decode_matches_reference_cfg1(golden_cfg1, cfg1_ensemble, precision, tag):
    g = golden_cfg1
    e = int(tag[1:]) / 1000
    cfg = DecoderConfig(precision=precision)
    dec, res = _decode_rows(cfg1_ensemble, g[f"{tag}_noisy"], g[f"{tag}_syn"], e, cfg,
                            flags=N.MBP_RECORD_HISTORY)
    assert np.array_equal(res.converged, g[f"{tag}_converged"])
    assert np.array_equal(res.iterations, g[f"{tag}_iterations"])
    assert np.array_equal(res.mismatches, g[f"{tag}_mismatches"])
    conv = g[f"{tag}_converged"]
    assert np.array_equal(res.corrected[conv], g[f"{tag}_corrected"][conv])
    for k in range(res.corrected.shape[0]):
        rows = int(g[f"{tag}_hist_rows"][k])
        hist = np.packbits(dec.history(k, rows), axis=1, bitorder="little")
        assert np.array_equal(hist, g[f"{tag}_history"][k, :rows]), k


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_posteriors_per_sweep_within_tolerance(golden_cfg1, cfg1_ensemble, precision):
    """Per-sweep posterior LLRs: decode with max_iterations=t and read the state."""
    g = golden_cfg1
    worst = 0.0
    for tag in ("e030", "e070", "e090"):
        P = g[f"{tag}_posterior"]
        e = int(tag[1:]) / 1000
        frames = P.shape[0]
        for t in range(1, P.shape[1]):
            cfg = DecoderConfig(max_iterations=t, precision=precision)
            dec, _ = _decode_rows(cfg1_ensemble, g[f"{tag}_noisy"][:frames], g[f"{tag}_syn"][:frames], e,
                                  cfg, flags=N.MBP_KEEP_STATE)
            for k in range(frames):
                if np.isnan(P[k, t, 0]):
                    continue
                worst = max(worst, rel_err(dec.posterior(k), P[k, t]))
    assert worst <= TOL[precision], worst


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_decoder_variants_match_reference(golden_mid, mid_ensemble, precision):
    """damping / isolated-per-matrix / clamp / max_iterations variants
    (decoder.py:53-68) on the mid ensemble (conftest.py:17-20)."""
    g = golden_mid
    report = []
    for vi, vname in enumerate(g["variants"]):
        max_it, clamp, damping, joint = g["variant_params"][vi]
        cfg = DecoderConfig(int(max_it), float(clamp), float(damping),
                            "joint-graph" if joint else "isolated-per-matrix", precision)
        for u in (1, 3):
            ens = mid_ensemble.prefix(u)
            for e in ("050", "080", "110", "300"):
                tag = f"{vname}_e{e}_u{u}"
                dec, res = _decode_rows(ens, g[f"{tag}_noisy"], g[f"{tag}_syn"], int(e) / 1000, cfg,
                                        flags=N.MBP_RECORD_HISTORY)
                ok_conv = np.array_equal(res.converged, g[f"{tag}_converged"])
                ok_it = np.array_equal(res.iterations, g[f"{tag}_iterations"])
                ok_mm = np.array_equal(res.mismatches, g[f"{tag}_mismatches"])
                hist_ok = True
                for k in range(res.corrected.shape[0]):
                    rows = int(g[f"{tag}_hist_rows"][k])
                    hist = np.packbits(dec.history(k, rows), axis=1, bitorder="little")
                    hist_ok &= np.array_equal(hist, g[f"{tag}_history"][k, :rows])
                if not (ok_conv and ok_it and ok_mm and hist_ok):
                    report.append((tag, ok_conv, ok_it, ok_mm, hist_ok))
    assert not report, report


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_u1_final_messages(golden_u1, precision):
    """test_equivalence.py:38-60 geometry through the drop-in decode()."""
    from paper_2001_07979_b200 import BitBlock, DecoderWorkspace, decode

    g = golden_u1
    h = ParityCheckMatrix._from_csr(256, 128, g["chk_ptr"], g["chk_var"])
    ens = MatrixEnsemble((h,))
    cfg = DecoderConfig(max_iterations=30, precision=precision)
    for s in range(3):
        t = f"s{s}"
        ws = DecoderWorkspace(ens, cfg)
        res = decode(ens, BitBlock(g[f"{t}_noisy"], 256), [BitBlock(g[f"{t}_syn"], 128)],
                     float(g[f"{t}_e"]), cfg, workspace=ws, track_decisions=True)
        assert res.converged == bool(g[f"{t}_converged"])
        assert res.iterations_used == int(g[f"{t}_iterations"])
        assert np.array_equal(res.decision_history, g[f"{t}_history"])
        for name in ("c2v", "v2c", "posterior"):
            assert rel_err(getattr(ws, name), g[f"{t}_{name}"]) <= TOL[precision], (t, name)


# ---------------------------------------------------------------------------
# full-size parity: cfg2 (n=65536, u=2) and cfg3 (u=3, m=14650)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name,tag", [("cfg2", "e020"), ("cfg2", "e030"), ("cfg2", "e050"), ("cfg3", "e030")])
def test_full_size_matches_reference(request, name, tag):
    g = request.getfixturevalue(f"golden_{name}")
    ens = request.getfixturevalue(f"{name}_ensemble")
    n = ens.n
    e = int(tag[1:]) / 1000
    frames = g[f"{tag}_converged"].shape[0]
    fb = make_frames(n, e, frames, seed=0)
    for k in range(frames):
        assert hashlib.sha256(fb.keys[k].tobytes()).hexdigest() == str(g[f"{tag}_key_sha"][k])
    dec = BatchDecoder(ens, frames)
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, e)
    assert np.array_equal(res.converged, g[f"{tag}_converged"])
    assert np.array_equal(res.iterations, g[f"{tag}_iterations"])
    assert np.array_equal(res.mismatches, g[f"{tag}_mismatches"])
    for k in range(frames):
        assert hashlib.sha256(res.corrected[k].tobytes()).hexdigest() == str(g[f"{tag}_corrected_sha"][k])


def test_converged_frames_satisfy_syndromes_full_size(cfg2_ensemble):
    """converged => H_l * corrected = z^l for all l (SPEC invariant), 256 frames."""
    fb = make_frames(cfg2_ensemble.n, 0.04, 256, seed=3)
    dec = BatchDecoder(cfg2_ensemble, 256)
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, 0.04)
    assert res.converged.mean() > 0.99
    resyn = dec.syndromes(res.corrected)
    assert np.array_equal(resyn[res.converged], syn[res.converged])
    assert np.all(res.mismatches[res.converged] == 0)
    # bit-exact recovery of Alice's key for every converged frame
    assert np.array_equal(res.corrected[res.converged], fb.keys[res.converged])


# ---------------------------------------------------------------------------
# batching, edge cases, determinism
# ---------------------------------------------------------------------------

def test_batch_composition_independent(golden_cfg1, cfg1_ensemble):
    g = golden_cfg1
    noisy, syn = g["e090_noisy"], g["e090_syn"]
    full = BatchDecoder(cfg1_ensemble, 32).decode(noisy, syn, 0.09)
    for lo, hi in ((0, 1), (3, 8), (5, 32)):
        part = BatchDecoder(cfg1_ensemble, 40).decode(noisy[lo:hi], syn[lo:hi], 0.09)
        assert np.array_equal(part.corrected, full.corrected[lo:hi])
        assert np.array_equal(part.iterations, full.iterations[lo:hi])
    # chunking: capacity smaller than the batch
    small = BatchDecoder(cfg1_ensemble, 5).decode(noisy, syn, 0.09)
    assert np.array_equal(small.corrected, full.corrected)
    assert np.array_equal(small.iterations, full.iterations)
    # per-frame e equals scalar e
    pf = BatchDecoder(cfg1_ensemble, 32).decode(noisy, syn, np.full(32, 0.09))
    assert np.array_equal(pf.iterations, full.iterations)


def test_zero_error_and_mixed_frames(golden_cfg1, cfg1_ensemble):
    g = golden_cfg1
    keys, syn = g["e030_key"][:33], g["e030_syn"][:33]
    dec = BatchDecoder(cfg1_ensemble, 33)
    res = dec.decode(keys, syn, 0.03)  # noisy == key: iteration 0 for all
    assert res.converged.all() and np.all(res.iterations == 0)
    assert np.array_equal(res.corrected, keys)
    mixed_noisy = g["e030_noisy"][:33].copy()
    mixed_noisy[::2] = keys[::2]
    res = dec.decode(mixed_noisy, syn, 0.03)
    assert np.all(res.iterations[::2] == 0)
    assert np.array_equal(res.iterations[1::2], g["e030_iterations"][1:33:2])


def test_failure_runs_to_limit(golden_mid, mid_ensemble):
    g = golden_mid
    cfg = DecoderConfig(max_iterations=40)
    res = BatchDecoder(mid_ensemble.prefix(1), 12, cfg).decode(g["default_e300_u1_noisy"], g["default_e300_u1_syn"], 0.3)
    assert not res.converged.any()
    assert np.all(res.iterations == 40)
    assert np.all(res.mismatches > 0)


def test_max_iterations_one_and_workspace_reuse(golden_cfg1, cfg1_ensemble):
    g = golden_cfg1
    dec = BatchDecoder(cfg1_ensemble, 32, DecoderConfig(max_iterations=1))
    r1 = dec.decode(g["e070_noisy"], g["e070_syn"], 0.07)
    assert np.all(r1.iterations <= 1)
    assert np.array_equal(r1.converged, g["e070_iterations"] <= 1)
    dec.configure(DecoderConfig())
    a = dec.decode(g["e070_noisy"], g["e070_syn"], 0.07)
    b = dec.decode(g["e070_noisy"], g["e070_syn"], 0.07)
    assert np.array_equal(a.corrected, b.corrected) and np.array_equal(a.iterations, g["e070_iterations"])


def test_joint_equals_stacked_decode(mid_ensemble):
    """Joint decode over H_1..H_u == decode of the stacked matrix (criterion 3)."""
    from paper_2001_07979_b200 import BitBlock, decode

    ens = mid_ensemble
    rows = [ens.matrices[l].row_adj(j) for l in range(ens.u) for j in range(ens.m)]
    # the stacked (u*m) x n matrix is wider than tall here, so decode it as an
    # ensemble of ONE matrix via a permissive constructor
    stacked = ParityCheckMatrix.__new__(ParityCheckMatrix)
    lay = stacked_layout(ens)
    ParityCheckMatrix.__init__(stacked, ens.n, ens.u * ens.m, lay.chk_ptr, lay.chk_var,
                               np.zeros(ens.n + 1, np.int64), np.zeros(0, np.int32))
    del rows
    fb = make_frames(ens.n, 0.07, 12, seed=9)
    dj = BatchDecoder(ens, 12, flags=N.MBP_RECORD_HISTORY)
    syn = dj.syndromes(fb.keys)
    rj = dj.decode(fb.noisy, syn, 0.07)
    # stacked single-matrix syndrome rows: bits concatenated without per-matrix padding
    bits = syn_bits_of(syn, ens.u, ens.m)
    ds = BatchDecoder(stacked, 12, flags=N.MBP_RECORD_HISTORY)
    rs = ds.decode(fb.noisy, pack_rows(bits), 0.07)
    assert np.array_equal(rj.iterations, rs.iterations)
    assert np.array_equal(rj.corrected, rs.corrected)
    for k in range(12):
        assert np.array_equal(dj.history(k, int(rj.iterations[k]) + 1), ds.history(k, int(rs.iterations[k]) + 1))


def test_device_tensor_path(golden_cfg1, cfg1_ensemble):
    import torch

    g = golden_cfg1
    dev = torch.device("cuda:0")
    noisy = torch.from_numpy(g["e070_noisy"]).to(dev)
    syn = torch.from_numpy(g["e070_syn"]).to(dev)
    dec = BatchDecoder(cfg1_ensemble, 32)
    corrected, conv, iters, mism = dec.decode(noisy, syn, 0.07)
    torch.cuda.synchronize()
    assert np.array_equal(iters.cpu().numpy(), g["e070_iterations"])
    assert np.array_equal(corrected.cpu().numpy()[g["e070_converged"]], g["e070_corrected"][g["e070_converged"]])
    keys = torch.from_numpy(g["e070_key"]).to(dev)
    assert np.array_equal(dec.syndromes(keys).cpu().numpy(), g["e070_syn"])


# ---------------------------------------------------------------------------
# frame compaction (decode.cuh) must be invisible in every output
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("variant", ["default", "damp25", "isolated", "fp64"])
def test_compaction_is_transparent(golden_mid, mid_ensemble, cfg1_ensemble, variant):
    cfgs = {"default": DecoderConfig(), "damp25": DecoderConfig(damping=0.25),
            "isolated": DecoderConfig(combining_mode="isolated-per-matrix"),
            "fp64": DecoderConfig(precision="fp64")}
    cfg = cfgs[variant]
    cases = []
    # mixed easy/hard frames: mid ensemble u=1 (failures run to the limit) and cfg1 at e=0.09
    g = golden_mid
    noisy = np.concatenate([g[f"default_e{e}_u1_noisy"] for e in ("050", "080", "110")])
    syn = np.concatenate([g[f"default_e{e}_u1_syn"] for e in ("050", "080", "110")])
    cases.append((mid_ensemble.prefix(1), noisy, syn, np.repeat([0.05, 0.08, 0.11], 12)))
    fb = make_frames(cfg1_ensemble.n, 0.09, 320, seed=11)
    dec0 = BatchDecoder(cfg1_ensemble, 320)
    cases.append((cfg1_ensemble, fb.noisy, dec0.syndromes(fb.keys), 0.09))
    compacted = 0
    for ens, nz, sy, e in cases:
        on = BatchDecoder(ens, nz.shape[0], cfg)
        off = BatchDecoder(ens, nz.shape[0], cfg, flags=N.MBP_NO_COMPACTION)
        a = on.decode(nz, sy, e)
        compacted += on.last_stats()[1] > 0
        b = off.decode(nz, sy, e)
        assert off.last_stats()[1] == 0
        assert np.array_equal(a.corrected, b.corrected)
        assert np.array_equal(a.converged, b.converged)
        assert np.array_equal(a.iterations, b.iterations)
        assert np.array_equal(a.mismatches, b.mismatches)
    assert compacted >= 1
