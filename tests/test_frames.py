"""The frame generator (csrc/frames.cuh) against the reference's frame streams.

The reference draws frame idx of a grid point with numpy's SeedSequence +
Philox (channel.rng_stream, channel.py:29-35; bench._frame_inputs,
bench.py:123-130).  ``channel.make_frames`` calls numpy exactly that way; the
library's generator restates the algorithms and must give the same bits:
host build here (no GPU), device build in the -m gpu test.
"""

import numpy as np
import pytest

from paper_2001_07979_b200.channel import entropy_words, frame_bits, make_frames, make_frames_native


def test_entropy_words_follow_numpy_coercion():
    assert entropy_words(0).tolist() == [0]
    assert entropy_words(0, 5, 0).tolist() == [0, 5, 0]
    assert entropy_words(2**32 + 7).tolist() == [7, 1]
    assert entropy_words(2**64 - 1).tolist() == [0xFFFFFFFF, 0xFFFFFFFF]
    with pytest.raises(ValueError):
        entropy_words(-1)


@pytest.mark.parametrize("n,e,seed,path,start,frames", [
    (4096, 0.03, 0, (), 0, 8),            # cfg 1 bench frames
    (65536, 0.03, 0, (), 1020, 3),        # cfg 2 bench frames across a 1024 boundary
    (4096, 0.07, 0, (7,), 0, 4),          # smoke() frames
    (1000, 0.09, 3, (2, 99), 5, 4),       # ragged n (not a multiple of 8 or 32), warm-up path
    (37, 0.25, 11, (1, 2, 3), 0, 6),      # tiny ragged n
    (8, 0.45, 2**33 + 1, (), 2**32 + 3, 2),   # multi-word seed and frame index
    (300, 1e-9, 1, (), 0, 3),             # almost no flips
])
def test_native_generator_equals_numpy_streams(n, e, seed, path, start, frames):
    ref = make_frames(n, e, frames, seed=seed, path=path, start=start)
    got = make_frames_native(n, e, frames, seed=seed, path=path, start=start, threads=3)
    assert np.array_equal(got.keys, ref.keys)
    assert np.array_equal(got.noisy, ref.noisy)


def test_native_generator_padding_bits_zero():
    got = make_frames_native(13, 0.3, 5, threads=2)
    assert np.all(got.keys[:, 1] >> 5 == 0) and np.all(got.noisy[:, 1] >> 5 == 0)


def test_native_generator_flip_rate_and_bits():
    kb, yb = frame_bits(65536, 0.05, 0, (12,))
    fb = make_frames_native(65536, 0.05, 1, path=(), start=12)
    assert np.array_equal(np.unpackbits(fb.keys[0], bitorder="little"), kb)
    assert np.array_equal(np.unpackbits(fb.noisy[0], bitorder="little"), yb)
    rate = float(np.mean(kb != yb))
    assert abs(rate - 0.05) < 5 * np.sqrt(0.05 * 0.95 / 65536)


def test_native_generator_rejects_bad_arguments():
    with pytest.raises(ValueError):
        make_frames_native(64, 0.5, 1)
    with pytest.raises(ValueError):
        make_frames_native(64, 0.1, 1, path=tuple(range(30)))
