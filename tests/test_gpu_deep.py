"""Deeper parity at the benched configurations.

* per-sweep posterior LLRs at full size (cfg 2 at e = 0.03 / 0.05, cfg 3 at
  e = 0.03) for both decode kernels, with frame compaction active, against
  the oracle (the reference's decode_loop restated in C) stopped after t
  sweeps: |d| <= 1e-4 * max(|ref|, 1);
* |L| > llr_clamp: sweep 1 reads the UNCLAMPED prior (_kernels.py:353-355),
  later sweeps clamp -- decisions, iterations and posteriors vs the oracle;
* the reference's known-answer tests of the fine-grained API
  (test_decoder.py:117-194) through the device kernels of
  c2v_update / v2c_update / soft_decision.
"""

import numpy as np
import pytest

import oracle
from paper_2001_07979_b200 import BatchDecoder, BitBlock, DecoderConfig, DecoderWorkspace
from paper_2001_07979_b200 import _native as N
from paper_2001_07979_b200.bits import unpack_rows
from paper_2001_07979_b200.channel import make_frames
from paper_2001_07979_b200.decoder import c2v_update, soft_decision, v2c_update
from paper_2001_07979_b200.matrix import MatrixEnsemble, ParityCheckMatrix, stacked_layout

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-4          # |d| <= TOL * max(|ref|, 1), DESIGN.md §4


def _err(got, ref):
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)))


def _syn_bits(rows, u, m):
    mb = (m + 7) // 8
    return np.concatenate([unpack_rows(rows[:, l * mb:(l + 1) * mb], m) for l in range(u)], axis=1)


def _per_sweep_check(ens, e, B, frames, flags, clamp=30.0, seed=0, max_t=None):
    """Decode B frames with max_iterations = t for t = 1..T and compare the
    posterior of each frame in `frames` with the oracle's after t sweeps.
    Returns (worst error, sweeps at which the batch compacted)."""
    fb = make_frames(ens.n, e, B, seed=seed)
    og = oracle.OracleGraph(stacked_layout(ens))
    full = BatchDecoder(ens, B, DecoderConfig(llr_clamp=clamp), flags=flags & ~N.MBP_KEEP_STATE)
    syn = full.syndromes(fb.keys)
    res = full.decode(fb.noisy, syn, e)
    pick = list(frames) if frames is not None else []
    # plus the slowest frames: the ones the compaction moves
    order = np.argsort(-res.iterations, kind="stable")
    pick += [int(k) for k in order[:4] if int(k) not in pick]
    T = max_t or int(min(res.iterations[pick].max(), 6))
    nb = unpack_rows(fb.noisy[pick], ens.n)
    sb = _syn_bits(syn[pick], ens.u, ens.m)
    worst, compacted = 0.0, []
    for t in range(1, T + 1):
        cfg = DecoderConfig(max_iterations=t, llr_clamp=clamp)
        dec = BatchDecoder(ens, B, cfg, flags=flags | N.MBP_KEEP_STATE)
        r = dec.decode(fb.noisy, syn, e)
        if dec.last_stats()[1]:
            compacted.append(t)
        for q, k in enumerate(pick):
            ref = oracle.decode(og, nb[q], sb[q], e, max_iterations=t, clamp=clamp)
            assert bool(r.converged[k]) == ref["converged"], (t, k)
            assert int(r.iterations[k]) == ref["iterations"], (t, k)
            assert int(r.mismatches[k]) == ref["mismatches"], (t, k)
            worst = max(worst, _err(dec.posterior(k), ref["posterior"]))
    return worst, compacted


@pytest.mark.parametrize("kernel", ["scatter", "explicit"])
@pytest.mark.parametrize("name,e", [("cfg2", 0.03), ("cfg2", 0.05), ("cfg3", 0.03)])
def test_posteriors_per_sweep_full_size(request, name, e, kernel):
    ens = request.getfixturevalue(f"{name}_ensemble")
    flags = N.MBP_EXPLICIT_MESSAGES if kernel == "explicit" else 0
    worst, compacted = _per_sweep_check(ens, e, 128, range(4), flags)
    assert worst <= TOL_F32, worst
    if (name, e) == ("cfg2", 0.03):
        # ~92 % of the frames stop after sweep 2: the batch compacts before
        # sweep 3, so the later posteriors come from the compacted layout
        assert compacted, "expected the batch to compact"


@pytest.mark.parametrize("kernel", ["scatter", "explicit"])
def test_prior_above_clamp(cfg1_ensemble, kernel):
    """clamp 2.0 < L = ln(0.97/0.03) = 3.476: sweep 1 uses the unclamped prior."""
    flags = N.MBP_EXPLICIT_MESSAGES if kernel == "explicit" else 0
    worst, _ = _per_sweep_check(cfg1_ensemble, 0.03, 64, range(6), flags, clamp=2.0, max_t=5)
    assert worst <= TOL_F32, worst
    # whole decodes to the limit, every frame
    fb = make_frames(cfg1_ensemble.n, 0.03, 64, seed=4)
    cfg = DecoderConfig(llr_clamp=2.0, max_iterations=25)
    dec = BatchDecoder(cfg1_ensemble, 64, cfg, flags=flags)
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, 0.03)
    og = oracle.OracleGraph(stacked_layout(cfg1_ensemble))
    nb = unpack_rows(fb.noisy, cfg1_ensemble.n)
    sb = _syn_bits(syn, cfg1_ensemble.u, cfg1_ensemble.m)
    for k in range(64):
        ref = oracle.decode(og, nb[k], sb[k], 0.03, max_iterations=25, clamp=2.0)
        assert bool(res.converged[k]) == ref["converged"], k
        assert int(res.iterations[k]) == ref["iterations"], k
        assert int(res.mismatches[k]) == ref["mismatches"], k


# ---------------------------------------------------------------------------
# the reference's known answers for the fine-grained API (test_decoder.py)
# ---------------------------------------------------------------------------

C2V_DEG3_2_MINUS1 = -0.7353256640555192   # 2*atanh(tanh(1.0)*tanh(-0.5)), test_decoder.py:25
REL = {"fp64": 1e-12, "fp32": 2e-6}


def _tiny():
    return ParityCheckMatrix.from_check_adjacency(3, 2, [np.array([0, 1]), np.array([1, 2])])


def _deg3():
    return ParityCheckMatrix.from_check_adjacency(4, 2, [np.array([0, 1, 2]), np.array([1, 2, 3])])


def _bits(*b):
    return BitBlock.from_bits(np.array(b, dtype=np.uint8))


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_kat_c2v_degree_two_identity_and_sign(precision):
    ws = DecoderWorkspace(MatrixEnsemble((_tiny(),)), DecoderConfig(precision=precision))
    for level in (0.8, -2.5):
        ws.v2c[:] = 0.0
        ws.v2c[0] = level
        c2v_update(ws, 0, _bits(0, 0))
        assert ws.c2v[1] == pytest.approx(level, rel=REL[precision])
        c2v_update(ws, 0, _bits(1, 0))
        assert ws.c2v[1] == pytest.approx(-level, rel=REL[precision])


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_kat_c2v_degree_three_value(precision):
    ws = DecoderWorkspace(MatrixEnsemble((_deg3(),)), DecoderConfig(precision=precision))
    ws.v2c[0], ws.v2c[1], ws.v2c[2] = 2.0, -1.0, 9.9
    c2v_update(ws, 0, _bits(0, 0))
    assert ws.c2v[2] == pytest.approx(C2V_DEG3_2_MINUS1, rel=REL[precision])
    c2v_update(ws, 0, _bits(1, 0))
    assert ws.c2v[2] == pytest.approx(-C2V_DEG3_2_MINUS1, rel=REL[precision])


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_kat_c2v_saturates_at_clamp(precision):
    ws = DecoderWorkspace(MatrixEnsemble((_tiny(),)), DecoderConfig(llr_clamp=12.0, precision=precision))
    ws.v2c[0] = 500.0
    c2v_update(ws, 0, _bits(0, 0))
    assert ws.c2v[1] == 12.0


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_kat_v2c_hand_sums(precision):
    tol = 1e-12 if precision == "fp64" else 1e-6
    ws = DecoderWorkspace(MatrixEnsemble((_tiny(),)), DecoderConfig(precision=precision))
    ws.priors[:] = (0.0, 0.2, 0.0)
    ws.c2v[1], ws.c2v[2] = 1.5, -0.5
    v2c_update(ws, 0)
    assert ws.v2c[1] == pytest.approx(-0.3, abs=tol)
    assert ws.v2c[2] == pytest.approx(1.7, abs=tol)
    ws2 = DecoderWorkspace(MatrixEnsemble((_tiny(),)), DecoderConfig(precision=precision))
    ws2.priors[:] = (0.7, 0.0, 0.0)
    ws2.c2v[0] = 2.2
    v2c_update(ws2, 0)
    assert ws2.v2c[0] == pytest.approx(0.7, abs=tol)     # degree-1 variable -> its prior


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_kat_soft_decision(precision):
    tol = 1e-12 if precision == "fp64" else 1e-6
    ws = DecoderWorkspace(MatrixEnsemble((_tiny(),)), DecoderConfig(precision=precision))
    ws.priors[:] = (0.5, -1.25, 2.0)
    assert np.array_equal(soft_decision(ws), ws.priors)
    h2 = ParityCheckMatrix.from_check_adjacency(3, 2, [np.array([0, 2]), np.array([0, 1])])
    ws = DecoderWorkspace(MatrixEnsemble((_tiny(), h2)), DecoderConfig(precision=precision))
    ws.priors[:] = (0.0, -0.3, 0.0)
    sl1 = ws.matrix_slice(1)
    ws.c2v[1], ws.c2v[2], ws.c2v[sl1.start + 3] = 0.4, 0.6, 0.5
    assert soft_decision(ws)[1] == pytest.approx(1.2, abs=tol)
