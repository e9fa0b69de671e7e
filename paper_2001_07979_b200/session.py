"""Bob-side session batch decode and verification tags.

The reference decodes a session's k key blocks one by one through a thread
pool, with a fresh ``DecoderWorkspace`` per block (``session._decode_block``,
session.py:305-319, called from ``bob_run``, session.py:385-420).  Here all k
blocks go to the GPU as ONE batched decode, and the per-block verification
tags are checked afterwards on the host:

    outcomes = decode_blocks(ensemble, noisy_blocks, syndromes, e, decoder,
                             tag_seeds=seeds, tags=tags, tag_width=64)

returns, per block, the same ``(result, status, verified, elapsed)`` tuple
``_decode_block`` returns, so ``bob_run``'s report / RESULT messages / digest
code is unchanged.  ``elapsed`` is the batch's decode
time split evenly over its blocks (the blocks are decoded together).

Tags restate ``protocol.block_tag`` / ``protocol.whole_key_digest``
(protocol.py:198-219): keyed BLAKE2b-64 over the little-endian block length
and the packed block bytes.  Hashing stays on the host (hashlib releases the
GIL; at ~1 GB/s per core it keeps up with the decoder on a few cores).
"""

from __future__ import annotations

import hashlib
import struct
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .bits import BitBlock
from .decoder import BatchDecoder, DecodeResult, _cfg_of

# protocol.py:47-49
RESULT_FAILED = 0
RESULT_SUCCESS = 1
RESULT_TAG_MISMATCH = 2

__all__ = ["RESULT_FAILED", "RESULT_SUCCESS", "RESULT_TAG_MISMATCH", "block_tag", "whole_key_digest",
           "decode_blocks", "bob_decode_key"]


def _block_bytes(block) -> tuple[int, bytes]:
    if isinstance(block, tuple):
        return block
    return int(block.length), bytes(np.asarray(block.data, dtype=np.uint8).tobytes())


def block_tag(block, seed: bytes) -> bytes:
    """64-bit keyed verification tag of one key block (protocol.py:198-208).
    ``block`` is a BitBlock or a (length_bits, packed_bytes) pair."""
    length, data = _block_bytes(block)
    h = hashlib.blake2b(digest_size=8, key=seed)
    h.update(struct.pack("<Q", length))
    h.update(data)
    return h.digest()


def whole_key_digest(blocks, succeeded) -> bytes:
    """Session-end digest over the successfully reconciled blocks
    (protocol.py:211-219)."""
    flags = np.array([1 if s else 0 for s in succeeded], dtype=np.uint8)
    h = hashlib.blake2b(digest_size=8)
    h.update(struct.pack("<I", len(blocks)))
    h.update(np.packbits(flags, bitorder="little").tobytes())
    for block, ok in zip(blocks, succeeded):
        if ok:
            h.update(_block_bytes(block)[1])
    return h.digest()


def _rows(blocks, nbytes: int) -> np.ndarray:
    if isinstance(blocks, np.ndarray):
        return np.ascontiguousarray(blocks, dtype=np.uint8)
    return np.stack([np.asarray(b.data, dtype=np.uint8)[:nbytes] for b in blocks])


def _syndrome_rows(syndromes, u: int, mbytes: int) -> np.ndarray:
    """list (per block) of u syndrome BitBlocks -> rows [k, u*ceil(m/8)]
    (the wire layout of protocol.pack_syndromes, protocol.py:137-143)."""
    if isinstance(syndromes, np.ndarray):
        return np.ascontiguousarray(syndromes, dtype=np.uint8)
    out = np.empty((len(syndromes), u * mbytes), dtype=np.uint8)
    for k, syn in enumerate(syndromes):
        if len(syn) != u:
            raise ValueError(f"expected {u} syndromes for u={u}, got {len(syn)}")
        for l, s in enumerate(syn):
            out[k, l * mbytes:(l + 1) * mbytes] = np.asarray(s.data, dtype=np.uint8)[:mbytes]
    return out


def decode_blocks(ensemble, noisy_blocks, syndromes, e, decoder=None, tag_seeds=None, tags=None,
                  tag_width: int = 64, batch_decoder: BatchDecoder | None = None, hash_workers: int = 4):
    """Batched ``_decode_block`` over all k blocks of a session.

    noisy_blocks: k BitBlocks of length n (or rows [k, ceil(n/8)]);
    syndromes: k lists of u BitBlocks (or rows [k, u*ceil(m/8)]);
    tag_seeds / tags: k seeds and k 8-byte tags when tag_width == 64.
    Returns a list of (DecodeResult, status, verified, elapsed_s)."""
    cfg = _cfg_of(decoder)
    dec = batch_decoder
    k = len(noisy_blocks)
    if k == 0:
        return []
    if dec is None or dec.max_frames < k or dec.config != cfg:
        dec = BatchDecoder(ensemble, k, cfg)
    n, m, u = dec.dev.n, dec.dev.m, dec.dev.u
    nbytes, mbytes = (n + 7) // 8, (m + 7) // 8
    noisy = _rows(noisy_blocks, nbytes)
    syn = _syndrome_rows(syndromes, u, mbytes)
    t0 = time.perf_counter()
    res = dec.decode(noisy, syn, e)
    elapsed = (time.perf_counter() - t0) / k
    if tag_width and (tag_seeds is None or tags is None):
        raise ValueError("tag_width > 0 needs tag_seeds and tags")

    def tag_ok(i):
        return block_tag((n, res.corrected[i].tobytes()), tag_seeds[i]) == tags[i]

    checked = {}
    todo = [i for i in range(k) if res.converged[i]] if tag_width else []
    if todo:
        with ThreadPoolExecutor(max_workers=max(1, hash_workers)) as pool:
            for i, ok in zip(todo, pool.map(tag_ok, todo)):
                checked[i] = ok
    out = []
    for i in range(k):
        result = DecodeResult(BitBlock(res.corrected[i].copy(), n), bool(res.converged[i]),
                              int(res.iterations[i]), int(res.mismatches[i]))
        if not result.converged:
            status, verified = RESULT_FAILED, (None if not tag_width else False)
        elif tag_width:
            ok = checked[i]
            status, verified = (RESULT_SUCCESS if ok else RESULT_TAG_MISMATCH), ok
        else:
            status, verified = RESULT_SUCCESS, None
        out.append((result, status, verified, elapsed))
    return out


def bob_decode_key(ensemble, noisy_key: BitBlock, syndromes, e, decoder=None, tag_seeds=None, tags=None,
                   tag_width: int = 64, batch_decoder: BatchDecoder | None = None):
    """Decode a whole sifted key of k*n bits block by block in one batch
    (``bob_run``'s decode loop, session.py:325-425, without the transport).
    Returns (corrected key BitBlock, per-block outcomes, whole-key digest)."""
    n = ensemble.n
    if noisy_key.length % n:
        raise ValueError(f"key length {noisy_key.length} not divisible by block length {n}")
    k = noisy_key.length // n
    bits = noisy_key.to_bits()
    blocks = [BitBlock.from_bits(bits[i * n:(i + 1) * n]) for i in range(k)]
    outcomes = decode_blocks(ensemble, blocks, syndromes, e, decoder, tag_seeds, tags, tag_width,
                             batch_decoder)
    out_blocks = [o[0].corrected for o in outcomes]
    succeeded = [o[0].converged and o[2] is not False for o in outcomes]
    digest = whole_key_digest(out_blocks, succeeded)
    key = BitBlock.from_bits(np.concatenate([b.to_bits() for b in out_blocks]))
    return key, outcomes, digest
