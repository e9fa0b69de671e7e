"""The committed cfg 4 ensemble (BASELINE configs[3]: n = 2^20, u = 2,
base_seed = 1), built by the device PEG (mbp_peg_build_device), against the
content hashes of the same ensemble built by the reference's own numba
build_ensemble (tests/golden/make_ensembles.py cfg4, ~7 h per matrix; hashes
recorded in tests/golden/cfg4_reference_hashes.json).  Host only."""

import json
from pathlib import Path

import pytest

from conftest import ENSEMBLES, GOLDEN

CACHE = ENSEMBLES / "cfg4_n1048576_m524288_u2_s1.npz"
REF = GOLDEN / "cfg4_reference_hashes.json"


@pytest.mark.skipif(not CACHE.exists(), reason="cfg4 cache not committed")
def test_cfg4_cache_loads_with_its_hashes():
    from paper_2001_07979_b200.matrix import load_ensemble

    ens = load_ensemble(CACHE)          # verifies the stored content hashes
    assert (ens.n, ens.m, ens.u) == (1 << 20, 1 << 19, 2)
    assert all(int(h.column_degrees().min()) == 3 == int(h.column_degrees().max()) for h in ens.matrices)


@pytest.mark.skipif(not (CACHE.exists() and REF.exists()), reason="reference hashes not recorded")
def test_cfg4_cache_equals_the_reference_build():
    from paper_2001_07979_b200.matrix import load_ensemble

    ref = json.loads(REF.read_text())
    assert load_ensemble(CACHE).content_hashes() == ref["content_hashes"]
