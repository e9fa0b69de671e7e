"""ctypes binding of oracle/mbp_oracle.c (test infrastructure only).

Every function mirrors one reference kernel; see mbp_oracle.c for the
file:line map.  Arrays are numpy; the graph is any object with the stacked
layout fields (``edge_off``, ``chk_ptr``, ``chk_var``, ``var_ptr``,
``var_edge``, ``n``, ``m``, ``u``) such as
``paper_2001_07979_b200.matrix.StackedLayout`` or the reference's
``DecoderWorkspace``.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "libmbp_oracle.so"

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class _Graph(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("m", C.c_int64), ("u", C.c_int32),
        ("edge_off", C.c_void_p), ("chk_ptr", C.c_void_p), ("chk_var", C.c_void_p),
        ("var_ptr", C.c_void_p), ("var_edge", C.c_void_p),
    ]


def build() -> Path:
    """Compile the oracle with its Makefile (gcc), output under oracle/build/."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.orc_syndrome.argtypes = [_u8p, _i64p, _i32p, C.c_int64, C.c_int64, _u8p]
        L.orc_c2v_pass.argtypes = [_f64p, _f64p, _i64p, _u8p, C.c_int64, C.c_int64,
                                   C.c_int64, C.c_double, _f64p]
        L.orc_v2c_pass.argtypes = [_f64p, _f64p, _i64p, _i64p, _f64p, C.c_int64,
                                   C.c_int64, C.c_int64, C.c_int, C.c_double, C.c_double]
        L.orc_posterior_pass.argtypes = [_f64p, _i64p, _i64p, _f64p, C.c_int64, _f64p]
        L.orc_mismatch_count.argtypes = [_u8p, _i64p, _i32p, _u8p, C.c_int64]
        L.orc_mismatch_count.restype = C.c_int64
        L.orc_prior_magnitude.argtypes = [C.c_double]
        L.orc_prior_magnitude.restype = C.c_double
        L.orc_decode.argtypes = [C.POINTER(_Graph), _u8p, _f64p, _f64p, _f64p, _f64p, _u8p,
                                 _f64p, C.c_int, C.c_double, C.c_double, C.c_int, _u8p,
                                 C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        L.orc_decode.restype = C.c_int
        L.orc_decode_batch.argtypes = [C.POINTER(_Graph), _u8p, _u8p, _f64p, C.c_int64,
                                       C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                       _u8p, _u8p, _i32p, _i64p]
        _LIB = L
    return _LIB


class OracleGraph:
    """Keeps the stacked arrays alive and exposes the C struct."""

    def __init__(self, layout):
        self.n, self.m, self.u = int(layout.n), int(layout.m), int(len(layout.edge_off) - 1)
        self.edge_off = np.ascontiguousarray(layout.edge_off, dtype=np.int64)
        self.chk_ptr = np.ascontiguousarray(layout.chk_ptr, dtype=np.int64)
        self.chk_var = np.ascontiguousarray(layout.chk_var, dtype=np.int32)
        self.var_ptr = np.ascontiguousarray(layout.var_ptr, dtype=np.int64)
        self.var_edge = np.ascontiguousarray(layout.var_edge, dtype=np.int64)
        self.E = int(self.edge_off[-1])
        self.dmax = max(int(np.diff(self.chk_ptr).max()), 1)
        self.struct = _Graph(self.n, self.m, self.u,
                             self.edge_off.ctypes.data, self.chk_ptr.ctypes.data,
                             self.chk_var.ctypes.data, self.var_ptr.ctypes.data,
                             self.var_edge.ctypes.data)


def _graph(layout) -> OracleGraph:
    return layout if isinstance(layout, OracleGraph) else OracleGraph(layout)


def prior_magnitude(e: float) -> float:
    return lib().orc_prior_magnitude(float(e))


def syndrome(chk_ptr, chk_var, bits, lo=0, hi=None) -> np.ndarray:
    chk_ptr = np.ascontiguousarray(chk_ptr, dtype=np.int64)
    hi = len(chk_ptr) - 1 if hi is None else hi
    out = np.zeros(hi - lo, dtype=np.uint8)
    lib().orc_syndrome(np.ascontiguousarray(bits, dtype=np.uint8), chk_ptr,
                       np.ascontiguousarray(chk_var, dtype=np.int32), lo, hi, out)
    return out


def mismatch_count(layout, bits, syn) -> int:
    g = _graph(layout)
    return int(lib().orc_mismatch_count(np.ascontiguousarray(bits, dtype=np.uint8), g.chk_ptr,
                                        g.chk_var, np.ascontiguousarray(syn, dtype=np.uint8),
                                        g.u * g.m))


def c2v_pass(layout, v2c, c2v, syn_bits, matrix_index, clamp):
    """In-place C2V of one matrix; ``syn_bits`` is that matrix's u8[m]."""
    g = _graph(layout)
    scratch = np.zeros(g.dmax, dtype=np.float64)
    lib().orc_c2v_pass(v2c, c2v, g.chk_ptr, np.ascontiguousarray(syn_bits, dtype=np.uint8),
                       matrix_index * g.m, (matrix_index + 1) * g.m, matrix_index * g.m,
                       float(clamp), scratch)


def v2c_pass(layout, v2c, c2v, priors, matrix_index, joint=True, damping=0.0, clamp=30.0):
    g = _graph(layout)
    lib().orc_v2c_pass(v2c, c2v, g.var_ptr, g.var_edge, priors, g.n,
                       int(g.edge_off[matrix_index]), int(g.edge_off[matrix_index + 1]),
                       int(bool(joint)), float(damping), float(clamp))


def posterior_pass(layout, c2v, priors) -> np.ndarray:
    g = _graph(layout)
    out = np.zeros(g.n, dtype=np.float64)
    lib().orc_posterior_pass(c2v, g.var_ptr, g.var_edge, priors, g.n, out)
    return out


def decode(layout, noisy_bits, syn_bits, e, max_iterations=60, clamp=30.0, damping=0.0,
           joint=True, record=False):
    """One frame through the restated decode_loop.  ``noisy_bits`` u8[n],
    ``syn_bits`` u8[u*m] (concatenated per matrix).  Returns a dict with the
    DecodeResult fields plus the final workspace arrays."""
    g = _graph(layout)
    noisy_bits = np.ascontiguousarray(noisy_bits, dtype=np.uint8)
    priors = (1.0 - 2.0 * noisy_bits.astype(np.float64)) * prior_magnitude(e)
    v2c = np.zeros(g.E); c2v = np.zeros(g.E)
    post = np.zeros(g.n); hard = np.zeros(g.n, dtype=np.uint8)
    scratch = np.zeros(g.dmax)
    hist = np.zeros(((max_iterations + 1) if record else 1, g.n if record else 1), dtype=np.uint8)
    it = C.c_int32(0); bad = C.c_int64(0)
    conv = lib().orc_decode(C.byref(g.struct), np.ascontiguousarray(syn_bits, dtype=np.uint8),
                            priors, v2c, c2v, post, hard, scratch, int(max_iterations),
                            float(clamp), float(damping), int(bool(joint)), hist, int(record),
                            C.byref(it), C.byref(bad))
    return {
        "converged": bool(conv), "iterations": int(it.value), "mismatches": int(bad.value),
        "hard": hard, "posterior": post, "v2c": v2c, "c2v": c2v, "priors": priors,
        "history": hist[: it.value + 1] if record else None,
    }


def decode_batch(layout, noisy_packed, syn_packed, e, max_iterations=60, clamp=30.0,
                 damping=0.0, joint=True, threads=None):
    """Batch of packed frames on POSIX threads (the CPU baseline)."""
    g = _graph(layout)
    noisy_packed = np.ascontiguousarray(noisy_packed, dtype=np.uint8)
    B = noisy_packed.shape[0]
    ev = np.ascontiguousarray(np.broadcast_to(np.asarray(e, dtype=np.float64), (B,)))
    corrected = np.zeros_like(noisy_packed)
    converged = np.zeros(B, dtype=np.uint8)
    iterations = np.zeros(B, dtype=np.int32)
    mismatches = np.zeros(B, dtype=np.int64)
    threads = threads or os.cpu_count() or 1
    lib().orc_decode_batch(C.byref(g.struct), noisy_packed,
                           np.ascontiguousarray(syn_packed, dtype=np.uint8), ev, B,
                           int(max_iterations), float(clamp), float(damping), int(bool(joint)),
                           int(threads), corrected, converged, iterations, mismatches)
    return corrected, converged.astype(bool), iterations, mismatches
