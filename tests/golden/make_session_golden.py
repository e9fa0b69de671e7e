"""Golden vectors for the session batch decode and verification tags,
produced by the REFERENCE (session._decode_block, protocol.block_tag,
protocol.whole_key_digest; session.py:305-319, protocol.py:198-219).

k = 24 blocks of the cfg-1 ensemble (n = 4096, u = 2) at e = 0.07: the key
and noisy blocks come from the reference's bench._frame_inputs; tag seeds are
fixed bytes; blocks 3 and 11 get a corrupted tag (-> RESULT_TAG_MISMATCH).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_session_golden.py
"""
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(OUT))
sys.path.insert(0, "/root/reference/pkg/src")

from make_golden import meta, ref_ensemble  # noqa: E402
from mmrecon import protocol, session  # noqa: E402  (reference)
from mmrecon.bench import _frame_inputs  # noqa: E402
from mmrecon.bits import BitBlock  # noqa: E402
from mmrecon.decoder import DecoderConfig  # noqa: E402


def main():
    ens = ref_ensemble("cfg1_n4096_m2048_u2_s1.npz")
    k, e = 24, 0.07
    cfg = SimpleNamespace(e=e, decoder=DecoderConfig(), tag_width=64)
    keys, noisy, syn, seeds, tags = [], [], [], [], []
    for i in range(k):
        key, nz, syns = _frame_inputs(ens, ens.u, e, 5, (i,))
        seed = bytes((7 * i + j) % 256 for j in range(16))
        tag = protocol.block_tag(key, seed)
        if i in (3, 11):
            tag = bytes(b ^ 0xFF for b in tag)
        keys.append(key.data.copy())
        noisy.append(nz.data.copy())
        syn.append(np.concatenate([s.data for s in syns]))
        seeds.append(np.frombuffer(seed, dtype=np.uint8))
        tags.append(np.frombuffer(tag, dtype=np.uint8))
    status, verified, iters, conv, corrected = [], [], [], [], []
    out_blocks = []
    for i in range(k):
        result, st, ver, _ = session._decode_block(
            ens, BitBlock(noisy[i], ens.n),
            [BitBlock(syn[i][l * ens.m // 8:(l + 1) * ens.m // 8], ens.m) for l in range(ens.u)],
            bytes(seeds[i]), bytes(tags[i]), cfg)
        status.append(st)
        verified.append(-1 if ver is None else int(ver))
        iters.append(result.iterations_used)
        conv.append(result.converged)
        corrected.append(result.corrected.data.copy())
        out_blocks.append(result.corrected)
    succeeded = [c and v != 0 for c, v in zip(conv, verified)]
    digest = protocol.whole_key_digest(out_blocks, succeeded)
    # standalone tag known answers (lengths not a multiple of 8)
    kat_blocks = [BitBlock.from_bits((np.arange(n) % 3 == 0).astype(np.uint8)) for n in (1, 13, 64, 100)]
    kat = [protocol.block_tag(b, b"\x01\x02" * 8) for b in kat_blocks]
    np.savez_compressed(
        OUT / "golden_session.npz",
        keys=np.stack(keys), noisy=np.stack(noisy), syn=np.stack(syn), seeds=np.stack(seeds),
        tags=np.stack(tags), status=np.array(status), verified=np.array(verified),
        iterations=np.array(iters), converged=np.array(conv), corrected=np.stack(corrected),
        digest=np.frombuffer(digest, dtype=np.uint8), e=e,
        kat_lengths=np.array([1, 13, 64, 100]), kat_tags=np.stack([np.frombuffer(t, np.uint8) for t in kat]),
        meta=str(meta()))
    print("status", status, "digest", digest.hex())


if __name__ == "__main__":
    main()
