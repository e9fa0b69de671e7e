"""The C-ABI library (CPU checks: no GPU needed, no compute calls)."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_2001_07979_b200 import _native as N
from paper_2001_07979_b200.build import LIB

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "mbp.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(mbp_[a-z0-9_]+)\s*\(", text)))


def test_library_built_and_loads():
    assert LIB.exists(), "run __graft_entry__.build() first"
    lib = N.load()
    assert lib.mbp_version().startswith(b"mbp_b200")


def test_exports_every_declared_symbol():
    decl = declared_symbols()
    assert set(decl) == set(N.EXPORTS), set(decl) ^ set(N.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mbp_[a-z0-9_]+)\b", out))
    missing = set(decl) - exported
    assert not missing, missing


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_errors_are_raised_not_swallowed():
    lib = N.load()
    import ctypes as C
    # invalid argument: null pointers -> MBP_EINVAL mapped to ValueError
    with pytest.raises(ValueError):
        N.check(lib.mbp_ensemble_create(0, 0, 1, None, None, 0, C.byref(C.c_void_p())))
    assert b"null" in lib.mbp_last_error()


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(N, "_LIB", None)
    with pytest.raises(N.MBPError, match="no CPU fallback"):
        N.load(tmp_path / "absent.so")
    monkeypatch.setattr(N, "_LIB", None)
    N.load()


def test_config_validation_messages():
    from paper_2001_07979_b200 import DecoderConfig

    for bad in (dict(max_iterations=0), dict(llr_clamp=0.0), dict(damping=1.5),
                dict(combining_mode="layered"), dict(precision="fp16")):
        with pytest.raises(ValueError):
            DecoderConfig(**bad)
