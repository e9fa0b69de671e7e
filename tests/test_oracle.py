"""Pin the CPU oracle (oracle/mbp_oracle.c) against the reference's own outputs.

The golden fixtures under tests/golden/ were produced by the reference package
itself (tests/golden/make_golden.py); the known-answer values are the frozen
mpmath constants of the reference tests (test_decoder.py:23-25, 117-194).
Only after these pass is the oracle trusted as the checker of the CUDA path.
"""

import hashlib
import math

import numpy as np
import pytest

import oracle
from paper_2001_07979_b200.bits import unpack_rows
from paper_2001_07979_b200.channel import make_frames
from paper_2001_07979_b200.matrix import ParityCheckMatrix, MatrixEnsemble, stacked_layout

PRIOR_MAG_E_0_03 = 3.4760986898352731     # ln(0.97/0.03), test_decoder.py:24
C2V_DEG3_2_MINUS1 = -0.7353256640555192   # 2*atanh(tanh(1)*tanh(-0.5)), test_decoder.py:25


def syn_bits_of(rows, u, m):
    """u8[B, u*ceil(m/8)] -> u8[B, u*m] (concatenated per matrix)."""
    mb = (m + 7) // 8
    return np.concatenate([unpack_rows(rows[:, l * mb:(l + 1) * mb], m) for l in range(u)], axis=1)


# ---------------------------------------------------------------------------
# known answers
# ---------------------------------------------------------------------------

def tiny():
    return ParityCheckMatrix.from_check_adjacency(3, 2, [[0, 1], [1, 2]])


def deg3():
    return ParityCheckMatrix.from_check_adjacency(4, 2, [[0, 1, 2], [1, 2, 3]])


def test_prior_magnitude_kat():
    assert oracle.prior_magnitude(0.03) == pytest.approx(PRIOR_MAG_E_0_03, rel=1e-15)


def test_c2v_degree3_kat():
    lay = stacked_layout(MatrixEnsemble((deg3(),)))
    v2c = np.zeros(lay.edges); c2v = np.zeros(lay.edges)
    v2c[0], v2c[1], v2c[2] = 2.0, -1.0, 9.9
    oracle.c2v_pass(lay, v2c, c2v, np.array([0, 0], np.uint8), 0, 30.0)
    assert c2v[2] == pytest.approx(C2V_DEG3_2_MINUS1, rel=1e-14)
    oracle.c2v_pass(lay, v2c, c2v, np.array([1, 0], np.uint8), 0, 30.0)
    assert c2v[2] == pytest.approx(-C2V_DEG3_2_MINUS1, rel=1e-14)


def test_c2v_degree2_identity_and_saturation():
    lay = stacked_layout(MatrixEnsemble((tiny(),)))
    for level in (0.8, -2.5):
        v2c = np.zeros(lay.edges); c2v = np.zeros(lay.edges)
        v2c[0] = level
        oracle.c2v_pass(lay, v2c, c2v, np.array([0, 0], np.uint8), 0, 30.0)
        assert c2v[1] == pytest.approx(level, rel=1e-12)
        oracle.c2v_pass(lay, v2c, c2v, np.array([1, 0], np.uint8), 0, 30.0)
        assert c2v[1] == pytest.approx(-level, rel=1e-12)
    v2c = np.zeros(lay.edges); c2v = np.zeros(lay.edges)
    v2c[0] = 500.0
    oracle.c2v_pass(lay, v2c, c2v, np.array([0, 0], np.uint8), 0, 12.0)
    assert c2v[1] == 12.0


def test_v2c_and_posterior_hand_sums():
    lay = stacked_layout(MatrixEnsemble((tiny(),)))
    priors = np.array([0.0, 0.2, 0.0])
    c2v = np.zeros(lay.edges); v2c = np.zeros(lay.edges)
    c2v[1], c2v[2] = 1.5, -0.5
    oracle.v2c_pass(lay, v2c, c2v, priors, 0)
    assert v2c[1] == pytest.approx(-0.3, abs=1e-12)
    assert v2c[2] == pytest.approx(1.7, abs=1e-12)
    h2 = ParityCheckMatrix.from_check_adjacency(3, 2, [[0, 2], [0, 1]])
    lay2 = stacked_layout(MatrixEnsemble((tiny(), h2)))
    c2v = np.zeros(lay2.edges)
    c2v[1], c2v[2], c2v[int(lay2.edge_off[1]) + 3] = 0.4, 0.6, 0.5
    post = oracle.posterior_pass(lay2, c2v, np.array([0.0, -0.3, 0.0]))
    assert post[1] == pytest.approx(1.2, abs=1e-12)


# ---------------------------------------------------------------------------
# golden frames: cfg1 (n=4096, u=2), every error rate
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("tag", ["e030", "e070", "e090", "e110"])
def test_oracle_matches_reference_cfg1(golden_cfg1, cfg1_ensemble, tag):
    g = golden_cfg1
    lay = stacked_layout(cfg1_ensemble)
    og = oracle.OracleGraph(lay)
    n, m, u = lay.n, lay.m, lay.u
    keys = unpack_rows(g[f"{tag}_key"], n)
    noisy = unpack_rows(g[f"{tag}_noisy"], n)
    syn = syn_bits_of(g[f"{tag}_syn"], u, m)
    e = int(tag[1:]) / 1000
    for k in range(keys.shape[0]):
        assert np.array_equal(oracle.syndrome(lay.chk_ptr, lay.chk_var, keys[k]), syn[k])
        r = oracle.decode(og, noisy[k], syn[k], e, record=True)
        assert r["converged"] == bool(g[f"{tag}_converged"][k])
        assert r["iterations"] == int(g[f"{tag}_iterations"][k])
        assert r["mismatches"] == int(g[f"{tag}_mismatches"][k])
        assert np.array_equal(np.packbits(r["hard"], bitorder="little"), g[f"{tag}_corrected"][k])
        rows = int(g[f"{tag}_hist_rows"][k])
        hist = np.packbits(r["history"], axis=1, bitorder="little")
        assert np.array_equal(hist, g[f"{tag}_history"][k, :rows])
    if f"{tag}_posterior" in g:
        P = g[f"{tag}_posterior"]
        for k in range(P.shape[0]):
            for t in range(1, P.shape[1]):
                if np.isnan(P[k, t, 0]):
                    break
                r = oracle.decode(og, noisy[k], syn[k], e, max_iterations=t)
                ref = P[k, t]
                assert np.max(np.abs(r["posterior"] - ref) / np.maximum(np.abs(ref), 1.0)) <= 1e-12


# ---------------------------------------------------------------------------
# golden frames: every DecoderConfig variant on the mid ensemble
# ---------------------------------------------------------------------------

def test_oracle_matches_reference_variants(golden_mid, mid_ensemble):
    g = golden_mid
    checked = 0
    for vi, vname in enumerate(g["variants"]):
        max_it, clamp, damping, joint = g["variant_params"][vi]
        for u in (1, 3):
            lay = stacked_layout(mid_ensemble.prefix(u))
            og = oracle.OracleGraph(lay)
            for e in ("050", "080", "110", "300"):
                tag = f"{vname}_e{e}_u{u}"
                noisy = unpack_rows(g[f"{tag}_noisy"], lay.n)
                syn = syn_bits_of(g[f"{tag}_syn"], u, lay.m)
                for k in range(noisy.shape[0]):
                    r = oracle.decode(og, noisy[k], syn[k], int(e) / 1000, int(max_it), clamp, damping,
                                      bool(joint), record=True)
                    assert r["converged"] == bool(g[f"{tag}_converged"][k]), tag
                    assert r["iterations"] == int(g[f"{tag}_iterations"][k]), tag
                    assert r["mismatches"] == int(g[f"{tag}_mismatches"][k]), tag
                    rows = int(g[f"{tag}_hist_rows"][k])
                    assert np.array_equal(np.packbits(r["history"], axis=1, bitorder="little"),
                                          g[f"{tag}_history"][k, :rows]), tag
                    if k == 0 and f"{tag}_ws_c2v" in g:
                        for name in ("posterior", "v2c", "c2v"):
                            ref = g[f"{tag}_ws_{name}"]
                            got = r[name] if r["iterations"] else (np.zeros_like(ref) if name != "v2c" else r["v2c"])
                            assert np.max(np.abs(got - ref)) <= 1e-9 * max(1.0, np.abs(ref).max()), (tag, name)
                    checked += 1
    assert checked == 6 * 2 * 4 * 12


def test_oracle_u1_message_exact(golden_u1):
    g = golden_u1
    h = ParityCheckMatrix._from_csr(256, 128, g["chk_ptr"], g["chk_var"])
    lay = stacked_layout(MatrixEnsemble((h,)))
    for s in range(3):
        t = f"s{s}"
        r = oracle.decode(lay, unpack_rows(g[f"{t}_noisy"][None], 256)[0],
                          unpack_rows(g[f"{t}_syn"][None], 128)[0], float(g[f"{t}_e"]),
                          max_iterations=30, record=True)
        assert r["converged"] == bool(g[f"{t}_converged"])
        assert r["iterations"] == int(g[f"{t}_iterations"])
        assert np.array_equal(r["history"], g[f"{t}_history"])
        assert np.array_equal(r["c2v"], g[f"{t}_c2v"])
        assert np.array_equal(r["v2c"], g[f"{t}_v2c"])


# ---------------------------------------------------------------------------
# full-size ensembles: frames regenerated from seeds (pins channel.rng_stream too)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name,tag,frames", [("cfg2", "e030", 6), ("cfg2", "e050", 4), ("cfg3", "e030", 4)])
def test_oracle_matches_reference_full_size(request, name, tag, frames):
    g = request.getfixturevalue(f"golden_{name}")
    ens = request.getfixturevalue(f"{name}_ensemble")
    lay = stacked_layout(ens)
    og = oracle.OracleGraph(lay)
    e = int(tag[1:]) / 1000
    fb = make_frames(lay.n, e, frames, seed=0)
    for k in range(frames):
        assert hashlib.sha256(fb.keys[k].tobytes()).hexdigest() == str(g[f"{tag}_key_sha"][k])
        key = unpack_rows(fb.keys[k][None], lay.n)[0]
        noisy = unpack_rows(fb.noisy[k][None], lay.n)[0]
        syn = oracle.syndrome(lay.chk_ptr, lay.chk_var, key)
        r = oracle.decode(og, noisy, syn, e)
        assert r["converged"] == bool(g[f"{tag}_converged"][k])
        assert r["iterations"] == int(g[f"{tag}_iterations"][k])
        corrected = np.packbits(r["hard"], bitorder="little")
        assert hashlib.sha256(corrected.tobytes()).hexdigest() == str(g[f"{tag}_corrected_sha"][k])


def test_oracle_batch_driver_matches_single(cfg1_ensemble, golden_cfg1):
    g = golden_cfg1
    lay = stacked_layout(cfg1_ensemble)
    corrected, conv, iters, mism = oracle.decode_batch(lay, g["e070_noisy"], g["e070_syn"], 0.07, threads=4)
    assert np.array_equal(corrected, g["e070_corrected"])
    assert np.array_equal(conv, g["e070_converged"])
    assert np.array_equal(iters, g["e070_iterations"])
    assert np.array_equal(mism, g["e070_mismatches"])


def test_binary_entropy_and_efficiency():
    from paper_2001_07979_b200.channel import binary_entropy, efficiency
    assert binary_entropy(0.5) == 1.0
    assert binary_entropy(0.1) == pytest.approx(0.4689955935892812, rel=1e-14)
    assert efficiency(1 << 15, 1 << 16, 0.1) == pytest.approx(1.0661, abs=1e-4)
    assert efficiency(14650, 65536, 0.03) == pytest.approx(1.14995, abs=1e-4)
    assert math.isclose(binary_entropy(0.3), binary_entropy(0.7))
