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
           "FrameBatch", "make_frames", "entropy_words", "make_frames_native", "make_frames_device"]


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


def entropy_words(*ints: int) -> np.ndarray:
    """SeedSequence entropy words of a tuple of non-negative ints (numpy's
    _coerce_to_uint32_array: little-endian uint32 words, 0 -> one zero word)."""
    words = []
    for x in ints:
        x = int(x)
        if x < 0:
            raise ValueError("expected non-negative integers")
        if x == 0:
            words.append(0)
        while x:
            words.append(x & 0xFFFFFFFF)
            x >>= 32
    return np.asarray(words, dtype=np.uint32)


def _frame_prefix(seed: int, path: tuple) -> np.ndarray:
    w = entropy_words(seed, *path)
    if w.size > 21:
        raise ValueError("seed + path exceed 21 entropy words")
    return np.ascontiguousarray(w)


def make_frames_native(n: int, e: float, frames: int, seed: int = 0, path: tuple = (),
                       start: int = 0, threads: int | None = None) -> FrameBatch:
    """make_frames through the library's generator on host threads
    (mbp_frames_generate; frames.cuh restates numpy's SeedSequence / Philox /
    integers / random, checked bit for bit against make_frames in tests)."""
    import os

    from . import _native as N

    nb = (n + 7) // 8
    keys = np.empty((frames, nb), dtype=np.uint8)
    noisy = np.empty((frames, nb), dtype=np.uint8)
    pre = _frame_prefix(seed, tuple(path))
    N.call("mbp_frames_generate", int(n), pre.ctypes.data, int(pre.size), int(start), int(frames), float(e),
           keys.ctypes.data, noisy.ctypes.data, int(threads or os.cpu_count() or 1))
    return FrameBatch(keys, noisy, n, e)


def make_frames_device(n: int, e: float, frames: int, seed: int = 0, path: tuple = (), start: int = 0,
                       device: int = 0, out=None, stream=None):
    """The same frames generated in HBM (mbp_frames_generate_device): returns
    (keys, noisy) uint8 CUDA tensors [frames, ceil(n/8)] on ``device``,
    enqueued on the current torch stream (or ``stream``)."""
    import ctypes as C

    import torch

    from . import _native as N

    nb = (n + 7) // 8
    dev = torch.device("cuda", device)
    keys, noisy = out if out is not None else (torch.empty((frames, nb), dtype=torch.uint8, device=dev),
                                               torch.empty((frames, nb), dtype=torch.uint8, device=dev))
    for t in (keys, noisy):
        if t.dtype != torch.uint8 or not t.is_cuda or not t.is_contiguous() or tuple(t.shape) != (frames, nb):
            raise ValueError(f"output rows must be contiguous uint8 CUDA tensors of shape {(frames, nb)}")
    pre = _frame_prefix(seed, tuple(path))
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    N.call("mbp_frames_generate_device", int(n), pre.ctypes.data, int(pre.size), int(start), int(frames),
           float(e), keys.data_ptr(), noisy.data_ptr(), C.c_void_p(s))
    return keys, noisy


def bsc_flips(n: int, e: float, seed: int) -> np.ndarray:
    """Error pattern of ``bsc_corrupt(key, ChannelModel(e, seed))``
    (channel.py:106-114): u8[n], 1 where the bit flips."""
    return (rng_stream(seed).random(n) < e).astype(np.uint8)
