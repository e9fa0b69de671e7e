"""The device PEG (csrc/peg_gpu.cu: each edge's BFS on the GPU, the tie-break
stream on the host) builds exactly the reference's matrices: content hashes
equal the committed ensembles that the reference's own build_ensemble made
(tests/golden/make_ensembles.py), including cfg 2 at n = 65536, and the host
restatement (csrc/peg.cpp) on irregular column profiles."""

import numpy as np
import pytest

from paper_2001_07979_b200.matrix import build_ensemble, peg_construct

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,n,m,u,seed", [
    ("toy", 64, 32, 3, 41), ("mid", 512, 256, 3, 91), ("cfg1", 4096, 2048, 2, 1),
    ("desk", 16384, 8192, 3, 1001), ("cfg2", 65536, 32768, 2, 1),
])
def test_device_peg_reproduces_reference_ensembles(name, n, m, u, seed):
    from conftest import _ens

    ref = _ens(name)
    ours = build_ensemble(n, m, 3, u, seed, device=0)
    assert ours.content_hashes() == ref.content_hashes()


@pytest.mark.parametrize("n,m,seed", [(300, 120, 5), (2000, 700, 9), (1500, 1000, 77)])
def test_device_peg_equals_host_peg_irregular(n, m, seed):
    rng = np.random.default_rng(seed)
    deg = rng.integers(2, 5, size=n).astype(np.int32)
    a = peg_construct(n, m, deg, seed=seed)
    b = peg_construct(n, m, deg, seed=seed, device=0)
    assert a.content_hash() == b.content_hash()


def test_staged_device_peg_equals_one_shot():
    """mbp_peg_build_device_range chained over [0, n) in uneven stages gives
    the one-shot matrix (the cfg 4 build checkpoints this way)."""
    from paper_2001_07979_b200.matrix import matrix_from_variable_rows, peg_device_stage

    n, m, seed = 4096, 2048, 1
    rows = np.full((n, 4), -1, dtype=np.int32)
    state = 0
    for lo, hi in ((0, 1000), (1000, 1001), (1001, 3333), (3333, n)):
        state = peg_device_stage(n, m, 3, seed, state, lo, hi, rows, 0)
    staged = matrix_from_variable_rows(n, m, rows)
    assert staged.content_hash() == peg_construct(n, m, 3, seed=seed).content_hash()
