"""B200-native multi-matrix belief-propagation (MBP) reconciliation decoder.

Drop-in for the decode path of the reference ``mmrecon`` package
(pkg/src/mmrecon/__init__.py:3-21): the same decoder names, data formats and
semantics, with syndrome computation and batched decoding running as
hand-written sm_100a CUDA kernels behind a C ABI (include/mbp.h).
"""

from .bits import BitBlock
from .channel import binary_entropy, efficiency, generate_key, make_frames, rng_stream
from .decoder import (
    BatchDecoder,
    BatchResult,
    DecodeResult,
    DecoderConfig,
    DecoderWorkspace,
    DeviceEnsemble,
    c2v_update,
    compute_syndrome,
    decode,
    decode_batch,
    init_priors,
    reset,
    soft_decision,
    syndrome_batch,
    v2c_update,
)
from .matrix import MatrixEnsemble, ParityCheckMatrix, code_rate, load_ensemble, stacked_layout

__version__ = "0.1.0"

__all__ = [
    "BitBlock", "binary_entropy", "efficiency", "generate_key", "make_frames", "rng_stream",
    "BatchDecoder", "BatchResult", "DecodeResult", "DecoderConfig", "DecoderWorkspace",
    "DeviceEnsemble", "c2v_update", "compute_syndrome", "decode", "decode_batch", "init_priors",
    "reset", "soft_decision", "syndrome_batch", "v2c_update",
    "MatrixEnsemble", "ParityCheckMatrix", "code_rate", "load_ensemble", "stacked_layout",
]
