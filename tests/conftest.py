import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
ENSEMBLES = ROOT / "paper_2001_07979_b200" / "ensembles"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with np.load(GOLDEN / name) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_cfg1():
    return load_golden("golden_cfg1.npz")


@pytest.fixture(scope="session")
def golden_mid():
    return load_golden("golden_mid.npz")


@pytest.fixture(scope="session")
def golden_u1():
    return load_golden("golden_u1.npz")


@pytest.fixture(scope="session")
def golden_cfg2():
    return load_golden("golden_cfg2.npz")


@pytest.fixture(scope="session")
def golden_cfg3():
    return load_golden("golden_cfg3.npz")


def _ens(name):
    from paper_2001_07979_b200.matrix import load_ensemble

    return load_ensemble(next(ENSEMBLES.glob(f"{name}_*.npz")))


@pytest.fixture(scope="session")
def cfg1_ensemble():
    return _ens("cfg1")


@pytest.fixture(scope="session")
def mid_ensemble():
    return _ens("mid")


@pytest.fixture(scope="session")
def toy_ensemble():
    return _ens("toy")


@pytest.fixture(scope="session")
def cfg2_ensemble():
    return _ens("cfg2")


@pytest.fixture(scope="session")
def cfg3_ensemble():
    return _ens("cfg3")
