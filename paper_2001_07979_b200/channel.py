"""BSC frame streams and the efficiency metric.

``rng_stream`` and ``frame_inputs`` reproduce the reference's counter-based
frame generator bit for bit (Philox keyed by SeedSequence((seed,)+path),
pkg/src/mmrecon/channel.py:29-35; bench._frame_inputs, bench.py:123-130), so
parity frames and bench frames are the ones the reference would decode.
``binary_entropy`` / ``efficiency`` restate channel.py:76-95.
"""

from __future__ import annotations

import math

import numpy as np

from .bits import BitBlock

__all__ = ["rng_stream", "binary_entropy", "efficiency", "generate_key", "frame_bits",
           "FrameBatch", "make_frames"]


def rng_stream(seed: int, *path: int) -> np.random.Generator:
    key = np.random.SeedSequence((seed,) + tuple(path)).generate_state(2, np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def binary_entropy(e: float) -> float:
    if not 0.0 <= e <= 1.0:
        raise ValueError(f"probability outside [0, 1]: {e}")
    if e in (0.0, 1.0):
        return 0.0
    return -e * math.log2(e) - (1.0 - e) * math.log2(1.0 - e)


def efficiency(m: int, n: int, e: float) -> float:
    if not 0.0 < e < 0.5:
        raise ValueError(f"crossover probability must be in (0, 0.5), got {e}")
    if not 0 < m < n:
        raise ValueError(f"need 0 < m < n, got m={m}, n={n}")
    return m / (n * binary_entropy(e))


def generate_key(length: int, seed: int) -> BitBlock:
    if length <= 0:
        raise ValueError(f"length must be positive, got {length}")
    return BitBlock.from_bits(rng_stream(seed).integers(0, 2, size=length, dtype=np.uint8))


def frame_bits(n: int, e: float, seed: int, path: tuple) -> tuple:
    """(key_bits u8[n], noisy_bits u8[n]) of frame ``path`` -- the two streams
    of bench._frame_inputs: (seed, *path, 0) for the key, (seed, *path, 1)
    for the flips."""
    key = rng_stream(seed, *path, 0).integers(0, 2, size=n, dtype=np.uint8)
    flips = (rng_stream(seed, *path, 1).random(n) < e).astype(np.uint8)
    return key, key ^ flips


class FrameBatch:
    """B frames as packed rows: keys, noisy keys (ceil(n/8) bytes each)."""

    def __init__(self, keys_packed: np.ndarray, noisy_packed: np.ndarray, n: int, e: float):
        self.keys = np.ascontiguousarray(keys_packed, dtype=np.uint8)
        self.noisy = np.ascontiguousarray(noisy_packed, dtype=np.uint8)
        self.n = int(n)
        self.e = float(e)

    @property
    def batch(self) -> int:
        return self.keys.shape[0]


def make_frames(n: int, e: float, frames: int, seed: int = 0, path: tuple = (),
                start: int = 0) -> FrameBatch:
    """Frames start..start+frames-1 of point ``path`` (frame i uses path+(i,)),
    the indexing of measure_throughput (bench.py:181-185)."""
    nb = (n + 7) // 8
    keys = np.empty((frames, nb), dtype=np.uint8)
    noisy = np.empty((frames, nb), dtype=np.uint8)
    for k in range(frames):
        kb, yb = frame_bits(n, e, seed, tuple(path) + (start + k,))
        keys[k] = np.packbits(kb, bitorder="little")
        noisy[k] = np.packbits(yb, bitorder="little")
    return FrameBatch(keys, noisy, n, e)


def bsc_flips(n: int, e: float, seed: int) -> np.ndarray:
    """Error pattern of ``bsc_corrupt(key, ChannelModel(e, seed))``
    (channel.py:106-114): u8[n], 1 where the bit flips."""
    return (rng_stream(seed).random(n) < e).astype(np.uint8)
