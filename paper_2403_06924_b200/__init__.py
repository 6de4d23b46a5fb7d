"""B200-native compensated INT8 GEMM (arXiv 2403.06924, "xigemm").

The hot path — quantize, INT8 tcgen05 GEMM, residual sparsification,
compensation GEMM with a fused epilogue — runs as hand-written sm_100a CUDA in
lib/libxigemm_b200.so behind the C-ABI in include/xigemm_c.h.  This package is
the Python mirror of the reference's API over that library.
"""
from ._lib import InvalidArgument, XgError, lib  # noqa: F401
from .api import *  # noqa: F401,F403

__version__ = "0.1.0"
