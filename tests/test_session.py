"""Session batch decode (paper_2001_07979_b200/session.py) against the
reference's own session._decode_block / protocol.block_tag /
protocol.whole_key_digest outputs (tests/golden/make_session_golden.py)."""

import numpy as np
import pytest

from paper_2001_07979_b200.bits import BitBlock
from paper_2001_07979_b200.session import (RESULT_FAILED, RESULT_SUCCESS, RESULT_TAG_MISMATCH, block_tag,
                                           bob_decode_key, decode_blocks, whole_key_digest)


@pytest.fixture(scope="module")
def gs():
    from conftest import load_golden

    return load_golden("golden_session.npz")


def test_block_tag_known_answers(gs):
    for length, tag in zip(gs["kat_lengths"], gs["kat_tags"]):
        b = BitBlock.from_bits((np.arange(int(length)) % 3 == 0).astype(np.uint8))
        assert block_tag(b, b"\x01\x02" * 8) == tag.tobytes()


def test_tags_and_digest_of_reference_session(gs):
    n = 4096
    for key, seed, tag, st in zip(gs["keys"], gs["seeds"], gs["tags"], gs["status"]):
        assert (block_tag(BitBlock(key, n), seed.tobytes()) == tag.tobytes()) == (st == RESULT_SUCCESS)
    blocks = [BitBlock(c, n) for c in gs["corrected"]]
    succeeded = [bool(c) and v != 0 for c, v in zip(gs["converged"], gs["verified"])]
    assert whole_key_digest(blocks, succeeded) == gs["digest"].tobytes()


def test_result_codes_match_protocol():
    assert (RESULT_FAILED, RESULT_SUCCESS, RESULT_TAG_MISMATCH) == (0, 1, 2)   # protocol.py:47-49


@pytest.mark.gpu
def test_decode_blocks_matches_reference_session(gs, cfg1_ensemble):
    n, m, u = 4096, 2048, 2
    noisy = [BitBlock(r, n) for r in gs["noisy"]]
    syn = [[BitBlock(r[l * m // 8:(l + 1) * m // 8], m) for l in range(u)] for r in gs["syn"]]
    seeds = [s.tobytes() for s in gs["seeds"]]
    tags = [t.tobytes() for t in gs["tags"]]
    out = decode_blocks(cfg1_ensemble, noisy, syn, float(gs["e"]), tag_seeds=seeds, tags=tags)
    for i, (res, st, ver, el) in enumerate(out):
        assert st == int(gs["status"][i]), i
        assert (-1 if ver is None else int(ver)) == int(gs["verified"][i]), i
        assert res.converged == bool(gs["converged"][i])
        assert res.iterations_used == int(gs["iterations"][i])
        assert np.array_equal(res.corrected.data, gs["corrected"][i])
        assert el >= 0
    # whole key through bob_decode_key: concatenated blocks, same digest
    key = BitBlock.from_bits(np.concatenate([b.to_bits() for b in noisy]))
    corrected, outcomes, digest = bob_decode_key(cfg1_ensemble, key, syn, float(gs["e"]), tag_seeds=seeds,
                                                 tags=tags)
    assert digest == gs["digest"].tobytes()
    assert corrected.length == len(noisy) * n
    assert [o[1] for o in outcomes] == [int(s) for s in gs["status"]]
