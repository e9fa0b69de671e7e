"""Parity of the production scatter decode kernel (csrc/scatter.cuh) with the
oracle (the reference's decode_loop restated in C) on configurations the
golden fixtures do not cover: per-frame crossover probabilities (a sweep-1
message table per frame), a clamp above the fp64 tanh saturation point (the
SAT code path), the explicit-message base of sweeps >= 4 with and without
frame compaction, the wide-row (degree 13/14, 128-register) instances, the
pipelined host path, and equality with the explicit-message kernel.

Bar: per frame `converged`, `iterations_used`,
`residual_syndrome_mismatches` equal to the oracle, corrected bits of
converged frames equal; posteriors within |d| <= 1e-4 * max(|ref|, 1).
"""

import os

import numpy as np
import pytest

import oracle
from paper_2001_07979_b200 import BatchDecoder, DecoderConfig
from paper_2001_07979_b200 import _native as N
from paper_2001_07979_b200.bits import unpack_rows
from paper_2001_07979_b200.channel import make_frames
from paper_2001_07979_b200.matrix import stacked_layout

pytestmark = pytest.mark.gpu


def _syn_bits(rows, u, m):
    mb = (m + 7) // 8
    return np.concatenate([unpack_rows(rows[:, l * mb:(l + 1) * mb], m) for l in range(u)], axis=1)


def _oracle_all(ens, noisy, syn, e, cfg, frames=None):
    lay = stacked_layout(ens)
    og = oracle.OracleGraph(lay)
    nb = unpack_rows(noisy, ens.n)
    sb = _syn_bits(syn, ens.u, ens.m)
    ev = np.broadcast_to(np.asarray(e, dtype=np.float64), (noisy.shape[0],))
    out = []
    for k in (range(noisy.shape[0]) if frames is None else frames):
        out.append(oracle.decode(og, nb[k], sb[k], float(ev[k]), max_iterations=cfg.max_iterations,
                                 clamp=cfg.llr_clamp, damping=cfg.damping,
                                 joint=cfg.combining_mode == "joint-graph"))
    return out


def _assert_matches(res, ref, frames=None):
    idx = list(range(len(ref))) if frames is None else list(frames)
    for r, k in zip(ref, idx):
        assert bool(res.converged[k]) == r["converged"], k
        assert int(res.iterations[k]) == r["iterations"], k
        assert int(res.mismatches[k]) == r["mismatches"], k
        if r["converged"]:
            assert np.array_equal(res.corrected[k], np.packbits(r["hard"], bitorder="little")), k


def test_per_frame_crossover_probabilities(cfg1_ensemble):
    """One e per frame: the prior and the sweep-1 message magnitudes differ
    per lane (decode with frames drawn at 3-9 % but decoded with their own e)."""
    rng = np.random.default_rng(21)
    B = 96
    es = rng.uniform(0.03, 0.09, size=B)
    fb = [make_frames(cfg1_ensemble.n, float(es[k]), 1, seed=100 + k) for k in range(B)]
    keys = np.concatenate([f.keys for f in fb])
    noisy = np.concatenate([f.noisy for f in fb])
    dec = BatchDecoder(cfg1_ensemble, B)
    syn = dec.syndromes(keys)
    res = dec.decode(noisy, syn, es)
    _assert_matches(res, _oracle_all(cfg1_ensemble, noisy, syn, es, DecoderConfig()))


@pytest.mark.parametrize("clamp", [40.0, 60.0])
def test_clamp_above_saturation(cfg1_ensemble, clamp):
    """llr_clamp >= the fp64 tanh saturation point (~38.1): inputs with
    |x| >= sat must act as t = 1 exactly (the SAT path of rule_sd)."""
    cfg = DecoderConfig(llr_clamp=clamp)
    fb = make_frames(cfg1_ensemble.n, 0.08, 64, seed=31)
    dec = BatchDecoder(cfg1_ensemble, 64, cfg)
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, 0.08)
    _assert_matches(res, _oracle_all(cfg1_ensemble, fb.noisy, syn, 0.08, cfg))


@pytest.mark.parametrize("compaction", [True, False])
def test_long_decodes_explicit_base(cfg1_ensemble, compaction):
    """e = 0.10 at R = 1/2, n = 4096: many frames need 4..60 sweeps (explicit
    c2v base from sweep 4), some fail; with and without compaction."""
    flags = 0 if compaction else N.MBP_NO_COMPACTION
    fb = make_frames(cfg1_ensemble.n, 0.10, 160, seed=41)
    dec = BatchDecoder(cfg1_ensemble, 160, flags=flags)
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, 0.10)
    assert res.iterations.max() >= 5
    _assert_matches(res, _oracle_all(cfg1_ensemble, fb.noisy, syn, 0.10, DecoderConfig()))


def test_scatter_equals_explicit_kernel(cfg1_ensemble):
    """Same decisions from the scatter kernel and the explicit-message kernel
    (both fp32); posteriors within the fp32 tolerance of each other."""
    fb = make_frames(cfg1_ensemble.n, 0.07, 64, seed=51)
    sc = BatchDecoder(cfg1_ensemble, 64)
    ex = BatchDecoder(cfg1_ensemble, 64, flags=N.MBP_EXPLICIT_MESSAGES)
    syn = sc.syndromes(fb.keys)
    a = sc.decode(fb.noisy, syn, 0.07)
    b = ex.decode(fb.noisy, syn, 0.07)
    for f in ("corrected", "converged", "iterations", "mismatches"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    for t in (1, 2, 3):
        cfg = DecoderConfig(max_iterations=t)
        s2 = BatchDecoder(cfg1_ensemble, 64, cfg, flags=N.MBP_KEEP_STATE)
        e2 = BatchDecoder(cfg1_ensemble, 64, cfg, flags=N.MBP_KEEP_STATE | N.MBP_EXPLICIT_MESSAGES)
        s2.decode(fb.noisy, syn, 0.07)
        e2.decode(fb.noisy, syn, 0.07)
        for k in (0, 13, 63):
            p, q = s2.posterior(k), e2.posterior(k)
            assert float(np.max(np.abs(p - q) / np.maximum(np.abs(q), 1.0))) <= 1e-4


def test_wide_rows_cfg3_with_saturation_path(cfg3_ensemble):
    """Degree 13/14 rows (the 128-register instance) through the generic
    (SAT) path: clamp 40, 32 frames, against the oracle."""
    cfg = DecoderConfig(llr_clamp=40.0)
    fb = make_frames(cfg3_ensemble.n, 0.03, 32, seed=61)
    dec = BatchDecoder(cfg3_ensemble, 32, cfg)
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, 0.03)
    frames = range(0, 32, 4)   # the oracle needs ~0.1 s per frame here
    _assert_matches(res, _oracle_all(cfg3_ensemble, fb.noisy, syn, 0.03, cfg, frames), frames)


@pytest.mark.parametrize("subbatches", ["1", "3", "8"])
def test_host_path_pipelining_is_transparent(cfg2_ensemble, subbatches):
    """mbp_decode_batch (host buffers) splits the batch into sub-batches whose
    copies overlap the decode; results equal the device-buffer path."""
    import torch

    B = 512
    fb = make_frames(cfg2_ensemble.n, 0.04, B, seed=71)
    dec = BatchDecoder(cfg2_ensemble, B)
    dev = torch.device("cuda:0")
    syn_d = dec.syndromes(torch.from_numpy(fb.keys).to(dev))
    ref = dec.decode_device(torch.from_numpy(fb.noisy).to(dev), syn_d, 0.04)
    torch.cuda.synchronize()
    old = os.environ.get("MBP_HOST_SUBBATCHES")
    os.environ["MBP_HOST_SUBBATCHES"] = subbatches
    try:
        res = dec.decode(fb.noisy, syn_d.cpu().numpy(), 0.04)
    finally:
        if old is None:
            del os.environ["MBP_HOST_SUBBATCHES"]
        else:
            os.environ["MBP_HOST_SUBBATCHES"] = old
    assert np.array_equal(res.corrected, ref[0].cpu().numpy())
    assert np.array_equal(res.converged, ref[1].cpu().numpy().astype(bool))
    assert np.array_equal(res.iterations, ref[2].cpu().numpy())
    assert np.array_equal(res.mismatches, ref[3].cpu().numpy())
    good = res.converged & np.all(res.corrected == fb.keys, axis=1)
    assert good.mean() > 0.99


@pytest.fixture(scope="module")
def cfg4_ensemble():
    """u = 2, n = 2^20, m = 2^19 (BASELINE configs[3], long-key frames whose
    messages far exceed shared memory and L2): the PEG cache built by the
    device PEG (build_ensemble(2^20, 2^19, 3, u=2, base_seed=1)) when it is
    committed, else synthetic random (3, 6)-regular graphs."""
    from conftest import ENSEMBLES
    from paper_2001_07979_b200.matrix import load_ensemble, random_regular_ensemble

    p = ENSEMBLES / "cfg4_n1048576_m524288_u2_s1.npz"
    return load_ensemble(p) if p.exists() else random_regular_ensemble(1 << 20, 1 << 19, 2, seed=7)


def test_long_key_cfg4_against_oracle(cfg4_ensemble):
    ens = cfg4_ensemble
    B = 8
    fb = make_frames(ens.n, 0.03, B, seed=91)
    dec = BatchDecoder(ens, B)
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, 0.03)
    assert res.converged.all()
    assert np.array_equal(res.corrected, fb.keys)           # Alice's key recovered bit for bit
    assert np.array_equal(dec.syndromes(res.corrected), syn)
    frames = (0, 5)
    _assert_matches(res, _oracle_all(ens, fb.noisy, syn, 0.03, DecoderConfig(), frames), frames)


def _random_ensemble(rng, u):
    """u random irregular matrices sharing (n, m): column degrees 1-4, row
    degrees whatever falls out (2..~30) -- exercises the padded / exact-degree
    row variants, the wide-row instances and the irregular sweep-1 path."""
    from paper_2001_07979_b200.matrix import MatrixEnsemble, ParityCheckMatrix

    n = int(rng.integers(64, 1500))
    m = int(rng.integers(max(8, n // 8), n // 2))
    mats = []
    while len(mats) < u:
        rows = [[] for _ in range(m)]
        for i in range(n):
            for c in rng.choice(m, size=int(rng.integers(1, 5)), replace=False):
                rows[int(c)].append(i)
        if any(not r for r in rows):
            continue
        mats.append(ParityCheckMatrix.from_check_adjacency(n, m, rows))
    return MatrixEnsemble(tuple(mats))


@pytest.mark.parametrize("seed", range(10))
def test_random_irregular_ensembles_against_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    ens = _random_ensemble(rng, int(rng.integers(1, 4)))
    e = float(rng.uniform(0.01, 0.08))
    clamp = float(rng.choice([8.0, 30.0, 45.0]))
    B = int(rng.integers(33, 100))
    cfg = DecoderConfig(max_iterations=int(rng.integers(5, 40)), llr_clamp=clamp)
    fb = make_frames(ens.n, e, B, seed=seed)
    dec = BatchDecoder(ens, B, cfg)
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, e)
    _assert_matches(res, _oracle_all(ens, fb.noisy, syn, e, cfg))


@pytest.mark.parametrize("variant", ["damping", "isolated", "fp64", "explicit"])
@pytest.mark.parametrize("seed", range(4))
def test_random_irregular_explicit_kernel_against_oracle(seed, variant):
    """The explicit-message kernel (fp64 parity mode, damping, isolated
    combining, MBP_EXPLICIT_MESSAGES) on the same random irregular ensembles."""
    rng = np.random.default_rng(2000 + seed)
    ens = _random_ensemble(rng, int(rng.integers(1, 4)))
    e = float(rng.uniform(0.01, 0.07))
    B = int(rng.integers(33, 70))
    kw = {"damping": dict(damping=0.3), "isolated": dict(combining_mode="isolated-per-matrix"),
          "fp64": dict(precision="fp64"), "explicit": {}}[variant]
    cfg = DecoderConfig(max_iterations=int(rng.integers(5, 30)), **kw)
    fb = make_frames(ens.n, e, B, seed=seed)
    flags = N.MBP_EXPLICIT_MESSAGES if variant == "explicit" else 0
    dec = BatchDecoder(ens, B, cfg, flags=flags)
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, e)
    _assert_matches(res, _oracle_all(ens, fb.noisy, syn, e, cfg))


@pytest.mark.parametrize("e", [0.004, 0.012])
def test_low_qber_early_compaction(cfg1_ensemble, e):
    """At low QBER most frames stop after iteration 0 or sweep 1, so frames
    are compacted at the start of sweep 2 (the rebuilt-base path in the
    compacted layout, absolute accumulation); outputs equal the uncompacted
    decode and the oracle."""
    fb = make_frames(cfg1_ensemble.n, e, 256, seed=101)
    on = BatchDecoder(cfg1_ensemble, 256)
    off = BatchDecoder(cfg1_ensemble, 256, flags=N.MBP_NO_COMPACTION)
    syn = on.syndromes(fb.keys)
    a = on.decode(fb.noisy, syn, e)
    b = off.decode(fb.noisy, syn, e)
    for f in ("corrected", "converged", "iterations", "mismatches"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert on.last_stats()[1] in (0, 2, 3)
    frames = list(range(0, 256, 16))
    _assert_matches(a, _oracle_all(cfg1_ensemble, fb.noisy, syn, e, DecoderConfig(), frames), frames)


@pytest.mark.parametrize("e", [1e-12, 0.45])
def test_extreme_crossover_probabilities(cfg1_ensemble, e):
    """Huge priors (e -> 0: the fixed-point scale shrinks) and near-zero
    priors (e -> 0.5: decoding fails to the limit) against the oracle."""
    cfg = DecoderConfig(max_iterations=12)
    fb = make_frames(cfg1_ensemble.n, min(e, 0.02), 40, seed=111)
    dec = BatchDecoder(cfg1_ensemble, 40, cfg)
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, e)
    frames = list(range(0, 40, 5))
    _assert_matches(res, _oracle_all(cfg1_ensemble, fb.noisy, syn, e, cfg, frames), frames)


def test_partially_live_groups_sweeps_2_3(cfg2_ensemble):
    """cfg 2 at e = 0.04: a few frames of each 32-frame group finish after
    sweep 2, the rest after sweep 3, so the sweep-3 check phase runs its fast
    path on partially live groups (dead lanes masked by a zero fixed-point
    scale, scatter.cuh sc_span); the finished frames' outputs must not move."""
    B = 64
    fb = make_frames(cfg2_ensemble.n, 0.04, B, seed=0)
    dec = BatchDecoder(cfg2_ensemble, B, flags=N.MBP_NO_COMPACTION)
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, 0.04)
    it = res.iterations.reshape(2, 32)
    assert any(set(row.tolist()) >= {2, 3} for row in it), it
    _assert_matches(res, _oracle_all(cfg2_ensemble, fb.noisy, syn, 0.04, DecoderConfig()))


def test_phase_timers_account_for_the_compaction(cfg2_ensemble):
    """MBP_PROFILE_PHASES stamps: with a compaction the phases (initial check,
    per-sweep check / variable / syndrome, compaction, tail) add up to the
    kernel's stamped span, and decisions are those of the unprofiled decode."""
    import torch

    B = 256
    fb = make_frames(cfg2_ensemble.n, 0.03, B, seed=5)
    dev = torch.device("cuda:0")
    dec = BatchDecoder(cfg2_ensemble, B, flags=N.MBP_PROFILE_PHASES)
    syn = dec.syndromes(torch.from_numpy(fb.keys).to(dev))
    out = dec.decode_device(torch.from_numpy(fb.noisy).to(dev), syn, 0.03)
    torch.cuda.synchronize()
    pt = dec.phase_times()
    assert dec.last_stats()[1] >= 2 and "compaction_ms" in pt, pt
    parts = (pt["syncheck0_ms"] + sum(pt["check_ms"]) + sum(pt["var_ms"]) + sum(pt["syncheck_ms"])
             + sum(pt["compaction_ms"].values()) + pt["tail_ms"])
    assert min(pt["check_ms"]) >= 0.0
    assert abs(parts - pt["total_ms"]) <= 0.02 * pt["total_ms"] + 1e-3, (parts, pt)
    ref = BatchDecoder(cfg2_ensemble, B).decode_device(torch.from_numpy(fb.noisy).to(dev), syn, 0.03)
    for a, b in zip(out, ref):
        assert torch.equal(a, b)


@pytest.mark.parametrize("mix", [False, True])
def test_compaction_rebuild_of_post1_is_transparent(cfg2_ensemble, mix):
    """n >= 16384: a compaction at the start of sweep 3 rebuilds post'_1 in
    the compacted layout from the moved mismatch words instead of moving it
    (scatter.cuh sc_recomp_post1); every output must equal the uncompacted
    decode's.  mix: every fourth frame at e = 0.065 (sweeps 4+ after the
    compaction, on the explicit base), per-frame crossover probabilities."""
    B = 512
    if mix:
        # every fourth frame at e = 0.065: each 32-frame group is mostly
        # decided after sweep 2, so the decode compacts at sweep 3
        fa = make_frames(cfg2_ensemble.n, 0.025, 3 * B // 4, seed=21)
        fb = make_frames(cfg2_ensemble.n, 0.065, B // 4, seed=22)
        hard = np.arange(B) % 4 == 3
        keys = np.empty((B,) + fa.keys.shape[1:], fa.keys.dtype)
        noisy = np.empty((B,) + fa.noisy.shape[1:], fa.noisy.dtype)
        keys[~hard], keys[hard], noisy[~hard], noisy[hard] = fa.keys, fb.keys, fa.noisy, fb.noisy
        e = np.where(hard, 0.065, 0.025)
    else:
        fa = make_frames(cfg2_ensemble.n, 0.03, B, seed=21)
        keys, noisy, e = fa.keys, fa.noisy, 0.03
    on = BatchDecoder(cfg2_ensemble, B)
    off = BatchDecoder(cfg2_ensemble, B, flags=N.MBP_NO_COMPACTION)
    syn = on.syndromes(keys)
    a = on.decode(noisy, syn, e)
    assert on.last_stats()[1] == 3, on.last_stats()   # compacted at the start of sweep 3
    b = off.decode(noisy, syn, e)
    assert off.last_stats()[1] == 0
    for f in ("corrected", "converged", "iterations", "mismatches"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    if mix:
        assert a.iterations.max() >= 4
