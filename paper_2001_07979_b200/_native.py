"""ctypes binding of libmbp_b200.so (include/mbp.h).

The product path: every decode / syndrome call of this package goes through
these functions into the CUDA library.  There is no CPU fallback -- if the
library is missing or no GPU is present the call raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .build import LIB

MBP_OK, MBP_EINVAL, MBP_ECUDA, MBP_EUNSUPPORTED, MBP_ENOMEM = range(5)
MBP_JOINT_GRAPH, MBP_ISOLATED_PER_MATRIX = 0, 1
MBP_FP32_PHI, MBP_FP64_TANH = 0, 1
MBP_RECORD_HISTORY, MBP_KEEP_STATE, MBP_PROFILE_PHASES, MBP_NO_COMPACTION = 1, 2, 4, 8
MBP_EXPLICIT_MESSAGES = 16

#: every symbol include/mbp.h declares (checked by tests/test_native_abi.py)
EXPORTS = (
    "mbp_last_error", "mbp_version", "mbp_device_count",
    "mbp_ensemble_create", "mbp_ensemble_destroy", "mbp_ensemble_get_info",
    "mbp_workspace_create", "mbp_workspace_destroy", "mbp_workspace_configure",
    "mbp_syndrome_batch_device", "mbp_syndrome_batch",
    "mbp_decode_batch_device", "mbp_decode_batch",
    "mbp_workspace_read_posterior", "mbp_workspace_read_c2v", "mbp_workspace_read_v2c",
    "mbp_workspace_read_history", "mbp_workspace_read_phase_times",
    "mbp_c2v_pass", "mbp_v2c_pass", "mbp_posterior_pass",
    "mbp_host_alloc", "mbp_host_free", "mbp_workspace_last_timing", "mbp_workspace_last_stats",
    "mbp_peg_build", "mbp_peg_build_device", "mbp_peg_build_device_range",
    "mbp_frames_generate_device", "mbp_frames_generate",
)


class DecoderConfigC(C.Structure):
    _fields_ = [
        ("max_iterations", C.c_int32), ("combining_mode", C.c_int32),
        ("precision", C.c_int32), ("flags", C.c_int32),
        ("llr_clamp", C.c_double), ("damping", C.c_double),
    ]


class EnsembleInfoC(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("m", C.c_int32), ("u", C.c_int32), ("edges", C.c_int64),
        ("max_check_degree", C.c_int32), ("max_var_degree", C.c_int32),
        ("device", C.c_int32), ("sm_count", C.c_int32),
    ]


class MBPError(RuntimeError):
    pass


_VP = C.c_void_p
_SIGS = {
    "mbp_last_error": ([], C.c_char_p),
    "mbp_version": ([], C.c_char_p),
    "mbp_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "mbp_ensemble_create": ([C.c_int32, C.c_int32, C.c_int32, _VP, _VP, C.c_int, C.POINTER(_VP)], C.c_int),
    "mbp_ensemble_destroy": ([_VP], C.c_int),
    "mbp_ensemble_get_info": ([_VP, C.POINTER(EnsembleInfoC)], C.c_int),
    "mbp_workspace_create": ([_VP, C.c_int32, C.POINTER(DecoderConfigC), C.POINTER(_VP)], C.c_int),
    "mbp_workspace_destroy": ([_VP], C.c_int),
    "mbp_workspace_configure": ([_VP, C.POINTER(DecoderConfigC)], C.c_int),
    "mbp_syndrome_batch_device": ([_VP, _VP, C.c_int64, _VP, _VP], C.c_int),
    "mbp_syndrome_batch": ([_VP, _VP, C.c_int64, _VP], C.c_int),
    "mbp_decode_batch_device": ([_VP, _VP, _VP, _VP, C.c_int32, C.c_int64, _VP, _VP, _VP, _VP, _VP], C.c_int),
    "mbp_decode_batch": ([_VP, _VP, _VP, _VP, C.c_int32, C.c_int64, _VP, _VP, _VP, _VP], C.c_int),
    "mbp_workspace_read_posterior": ([_VP, C.c_int64, _VP], C.c_int),
    "mbp_workspace_read_c2v": ([_VP, C.c_int64, _VP], C.c_int),
    "mbp_workspace_read_v2c": ([_VP, C.c_int64, _VP], C.c_int),
    "mbp_workspace_read_history": ([_VP, C.c_int64, C.c_int32, _VP], C.c_int),
    "mbp_workspace_read_phase_times": ([_VP, _VP, C.c_int32, C.POINTER(C.c_int32)], C.c_int),
    "mbp_c2v_pass": ([_VP, C.c_int32, C.c_int32, _VP, C.c_double, _VP, _VP], C.c_int),
    "mbp_v2c_pass": ([_VP, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double, _VP, _VP, _VP], C.c_int),
    "mbp_posterior_pass": ([_VP, C.c_int32, _VP, _VP, _VP], C.c_int),
    "mbp_host_alloc": ([C.c_size_t], _VP),
    "mbp_peg_build": ([C.c_int32, C.c_int32, _VP, C.c_uint64, _VP, _VP], C.c_int),
    "mbp_peg_build_device": ([C.c_int32, C.c_int32, _VP, C.c_uint64, _VP, _VP, C.c_int], C.c_int),
    "mbp_peg_build_device_range": ([C.c_int32, C.c_int32, _VP, C.c_uint64, C.POINTER(C.c_uint64), C.c_int32,
                                    C.c_int32, _VP, C.c_int], C.c_int),
    "mbp_host_free": ([_VP], None),
    "mbp_frames_generate_device": ([C.c_int32, _VP, C.c_int32, C.c_int64, C.c_int64, C.c_double, _VP, _VP, _VP],
                                   C.c_int),
    "mbp_frames_generate": ([C.c_int32, _VP, C.c_int32, C.c_int64, C.c_int64, C.c_double, _VP, _VP, C.c_int32],
                            C.c_int),
    "mbp_workspace_last_timing": ([_VP, C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_int32)], C.c_int),
    "mbp_workspace_last_stats": ([_VP, C.POINTER(C.c_int32), C.POINTER(C.c_int32)], C.c_int),
}

_LIB = None


def load(path: Path | None = None) -> C.CDLL:
    """Load (never build) the library; raises if it is missing."""
    global _LIB
    if _LIB is None:
        p = Path(path or os.environ.get("MBP_LIB") or LIB)
        if not p.exists():
            raise MBPError(f"{p} not built: run `python -m paper_2001_07979_b200.build` "
                           "(the decoder has no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _LIB = lib
    return _LIB


def check(rc: int) -> None:
    if rc == MBP_OK:
        return
    msg = load().mbp_last_error().decode(errors="replace")
    if rc in (MBP_EINVAL, MBP_EUNSUPPORTED):
        raise ValueError(msg)
    if rc == MBP_ENOMEM:
        raise MemoryError(msg)
    raise MBPError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def ptr(a) -> int:
    """Data pointer of a numpy array or a torch tensor."""
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def device_count() -> int:
    n = C.c_int(0)
    call("mbp_device_count", C.byref(n))
    return n.value
