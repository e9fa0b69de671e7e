"""CPU oracle for the MBP decode path -- TEST INFRASTRUCTURE ONLY.

Checker for the CUDA product and the CPU baseline of bench.py; nothing under
``paper_2001_07979_b200/`` imports this package.  ``mbp_oracle.c`` restates the
reference's numba kernels (pkg/src/mmrecon/_kernels.py:220-379) in C/libm
double precision; this module binds it with ctypes.  Pinned against golden
vectors produced by the reference itself (tests/golden/, tests/test_oracle.py).
"""

from .oracle import (  # noqa: F401
    OracleGraph,
    build,
    c2v_pass,
    decode,
    decode_batch,
    lib,
    mismatch_count,
    posterior_pass,
    prior_magnitude,
    syndrome,
    v2c_pass,
)
