"""PEG construction (csrc/peg.cpp) reproduces the
reference's matrices exactly: the cached ensembles under
paper_2001_07979_b200/ensembles/ were built by the reference's own
build_ensemble (tests/golden/make_ensembles.py); content hashes
(matrix.py:106-113 in both packages) must match.  Host code: runs on CPU."""

import numpy as np
import pytest

from paper_2001_07979_b200.matrix import build_ensemble, peg_construct


@pytest.mark.parametrize("name,n,m,u,seed", [
    ("toy", 64, 32, 3, 41), ("mid", 512, 256, 3, 91), ("cfg1", 4096, 2048, 2, 1), ("desk", 16384, 8192, 3, 1001),
])
def test_peg_reproduces_reference_ensembles(name, n, m, u, seed):
    from conftest import _ens

    ref = _ens(name)
    ours = build_ensemble(n, m, 3, u, seed)
    assert ours.content_hashes() == ref.content_hashes()


def test_peg_invariants_and_validation():
    h = peg_construct(300, 120, np.r_[np.full(150, 2), np.full(150, 4)].astype(np.int32), seed=5)
    assert np.array_equal(h.column_degrees(), np.r_[np.full(150, 2), np.full(150, 4)])
    rows = [h.row_adj(j) for j in range(h.m)]
    assert all(np.all(np.diff(r) > 0) for r in rows)          # sorted, no parallel edges
    assert peg_construct(300, 120, 3, seed=5).content_hash() == peg_construct(300, 120, 3, seed=5).content_hash()
    assert peg_construct(300, 120, 3, seed=5).content_hash() != peg_construct(300, 120, 3, seed=6).content_hash()
    with pytest.raises(ValueError, match="column degree"):
        peg_construct(10, 5, 1, seed=0)
    with pytest.raises(ValueError, match="exceeds m"):
        peg_construct(10, 3, 4, seed=0)
