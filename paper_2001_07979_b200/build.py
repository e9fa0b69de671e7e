"""Build libmbp_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2001_07979_b200.build [--force]

The kernel template instances are split over several translation units
(csrc/k_*.cu) that compile in parallel; mbp.cu holds the host code and the
C ABI.  The shared library lands in paper_2001_07979_b200/_lib/ (git-ignored,
but it travels to the GPU box with the gpurun snapshot).  cudart is linked
statically so the .so depends only on the driver.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
OBJ_DIR = LIB_DIR / "obj"
LIB = LIB_DIR / "libmbp_b200.so"
# (object name, source, extra defines)
UNITS = [
    ("mbp", "mbp.cu", []),
    ("peg", "peg.cpp", []),
    ("frames", "frames.cu", []),
    ("peg_gpu", "peg_gpu.cu", []),
    ("k_explicit_f32", "k_explicit.cu", []),
    ("k_explicit_f64", "k_explicit.cu", ["-DMBP_EXPLICIT_F64=1"]),
    ("k_explicit_f64w", "k_explicit.cu", ["-DMBP_EXPLICIT_F64=2"]),
    ("k_scatter_0", "k_scatter.cu", ["-DMBP_SCATTER_PART=0"]),
    ("k_scatter_1", "k_scatter.cu", ["-DMBP_SCATTER_PART=1"]),
    ("k_scatter_2", "k_scatter.cu", ["-DMBP_SCATTER_PART=2"]),
]
DEPS = (sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cpp"))
        + [ROOT / "include" / "mbp.h"])

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-I", str(ROOT / "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libmbp_b200.so")


def source_hash() -> str:
    """SHA-256 (16 hex) over the library's sources and build flags: keys
    measurements (ncu DRAM traffic, profiles/decode_traffic.json) to the code
    they were taken on."""
    import hashlib

    h = hashlib.sha256(" ".join(NVCC_FLAGS[:-2]).encode())
    for p in DEPS:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()[:16]


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False, defines=(),
          out: Path | None = None) -> Path:
    """Compile the units in parallel and link; ``defines``/``out`` build a
    variant library elsewhere (experiments, e.g. MBP_SCATTER_MIN_BLOCKS=3)."""
    lib = Path(out) if out else LIB
    obj_dir = lib.parent / "obj"
    if not force and not out and not stale():
        return LIB
    obj_dir.mkdir(parents=True, exist_ok=True)
    cc = nvcc()

    headers = sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [ROOT / "include" / "mbp.h"]
    flags_file = obj_dir / "flags.txt"
    flags_now = " ".join([*NVCC_FLAGS, *[f"-D{d}" for d in defines], str(ptxas_info)])
    same_flags = flags_file.exists() and flags_file.read_text() == flags_now

    def compile_unit(unit):
        name, src, defs = unit
        obj = obj_dir / f"{name}.o"
        if not force and same_flags and obj.exists():
            t = obj.stat().st_mtime
            if all(p.stat().st_mtime <= t for p in [CSRC / src, *headers]):
                return obj   # up to date: sources and headers older than the object
        cmd = [cc, *NVCC_FLAGS, *defs, *[f"-D{d}" for d in defines], *(["-Xptxas", "-v"] if ptxas_info else []),
               "-c", "-o", str(obj),
               str(CSRC / src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src} {defs}:\n{r.stderr}")
        if ptxas_info or verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(UNITS)) as pool:
        objs = list(pool.map(compile_unit, UNITS))
    flags_file.write_text(flags_now)
    tmp = lib.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    tmp.replace(lib)
    return lib


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--ptxas", action="store_true")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    ap.add_argument("--out")
    a = ap.parse_args()
    print(build(force=a.force, verbose=True, ptxas_info=a.ptxas, defines=a.defines, out=a.out))
