"""Host-side data formats on the boundary (no GPU)."""

import hashlib

import numpy as np
import pytest

from paper_2001_07979_b200.bits import BitBlock, pack_rows, unpack_rows
from paper_2001_07979_b200.channel import bsc_flips, frame_bits, generate_key, make_frames, rng_stream
from paper_2001_07979_b200.decoder import init_priors
from paper_2001_07979_b200.matrix import (MatrixEnsemble, ParityCheckMatrix, load_ensemble, save_ensemble,
                                          stacked_layout)


def test_bitblock_roundtrip_and_padding():
    rng = np.random.default_rng(1)
    for n in (1, 7, 8, 9, 4096, 14650):
        bits = rng.integers(0, 2, n, dtype=np.uint8)
        b = BitBlock.from_bits(bits)
        assert np.array_equal(b.to_bits(), bits)
        assert b.weight() == int(bits.sum())
        assert all(b[i] == bits[i] for i in (0, n - 1))
    with pytest.raises(ValueError, match="padding"):
        BitBlock(np.array([0xFF], np.uint8), 3)
    rows = rng.integers(0, 2, (5, 37), dtype=np.uint8)
    assert np.array_equal(unpack_rows(pack_rows(rows), 37), rows)


def test_frames_match_reference_streams(golden_cfg1):
    """channel.frame_bits reproduces bench._frame_inputs (Philox/SeedSequence)."""
    fb = make_frames(4096, 0.07, 32, seed=0)
    assert np.array_equal(fb.keys, golden_cfg1["e070_key"])
    assert np.array_equal(fb.noisy, golden_cfg1["e070_noisy"])


def test_u1_frames_match_reference_helpers(golden_u1):
    key = generate_key(256, seed=1)
    assert np.array_equal(key.data, golden_u1["s1_key"])
    noisy = key.to_bits() ^ bsc_flips(256, 0.09, 50_001)
    assert np.array_equal(np.packbits(noisy, bitorder="little"), golden_u1["s1_noisy"])


def test_ensemble_cache_hashes(cfg1_ensemble, tmp_path):
    hashes = cfg1_ensemble.content_hashes()
    path = tmp_path / "e.npz"
    save_ensemble(cfg1_ensemble, path)
    assert load_ensemble(path).content_hashes() == hashes
    assert all(np.all(h.column_degrees() == 3) for h in cfg1_ensemble.matrices)


def test_stacked_layout_matches_reference_rules(mid_ensemble):
    lay = stacked_layout(mid_ensemble)
    assert lay.edges == 3 * mid_ensemble.n * mid_ensemble.u
    # matrix 0's edges first; var_edge ascending per variable
    for i in range(0, mid_ensemble.n, 37):
        ev = lay.var_edge[lay.var_ptr[i]:lay.var_ptr[i + 1]]
        assert np.all(np.diff(ev) > 0)
        assert np.all(lay.chk_var[ev] == i)
    assert lay.edge_off[1] == mid_ensemble.matrices[0].edge_count


def test_matrix_validation():
    with pytest.raises(ValueError, match="parallel edge"):
        ParityCheckMatrix.from_check_adjacency(4, 2, [[0, 0], [1, 2, 3]])
    with pytest.raises(ValueError, match="degree 0"):
        ParityCheckMatrix.from_check_adjacency(4, 2, [[0, 1], [1, 2]])
    h = ParityCheckMatrix.from_check_adjacency(3, 2, [[0, 1], [1, 2]])
    with pytest.raises(ValueError, match="identical"):
        MatrixEnsemble((h, h))


def test_init_priors_kat():
    pri = init_priors(BitBlock.from_bits(np.array([0, 1], np.uint8)), 0.03)
    assert pri[0] == pytest.approx(3.4760986898352731, rel=1e-14) and pri[0] == -pri[1]
    with pytest.raises(ValueError):
        init_priors(BitBlock.zeros(4), 0.5)


def test_rng_stream_is_path_keyed():
    a = rng_stream(0, 1, 2).integers(0, 1 << 30, 4)
    b = rng_stream(0, 1, 2).integers(0, 1 << 30, 4)
    c = rng_stream(0, 2, 1).integers(0, 1 << 30, 4)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    k, y = frame_bits(64, 0.5, 3, (1,))
    assert hashlib.sha256(k.tobytes()).hexdigest() != hashlib.sha256(y.tobytes()).hexdigest()
