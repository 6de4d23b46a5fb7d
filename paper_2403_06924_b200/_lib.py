"""ctypes binding of libxigemm_b200.so (the C-ABI in include/xigemm_c.h).

The library is built in-tree by paper_2403_06924_b200.build.  There is no
fallback: if the shared object is missing or no sm_100 device is present, the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
# XG_LIB_PATH: load another build of the library (A/B timing aid)
LIB_PATH = os.environ.get("XG_LIB_PATH") or os.path.join(PKG, "lib", "libxigemm_b200.so")


class XgError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    """Mirrors the reference's std::invalid_argument."""


class ShardRetry(XgError):
    """XG_EAGAIN from xg_shard_finish: the row-sharded run flagged more exact
    column means than its exchange buffer holds (`needed`); rerun with more."""

    def __init__(self, msg: str, needed: int = 0):
        super().__init__(msg)
        self.needed = needed


class XgConfig(C.Structure):
    _fields_ = [("bits", C.c_int), ("threshold", C.c_double), ("density_limit", C.c_double),
                ("scheme", C.c_int), ("policy", C.c_int), ("rounding", C.c_int)]


class XgReport(C.Structure):
    _fields_ = [("density_a", C.c_double), ("density_b", C.c_double), ("path", C.c_int),
                ("nnz_a", C.c_int64), ("nnz_b", C.c_int64), ("ns_quant", C.c_double),
                ("ns_xxmm", C.c_double), ("ns_reduce", C.c_double), ("ns_package", C.c_double),
                ("stats_fallbacks", C.c_int), ("ns_gemm_df", C.c_double),
                ("ns_gemm_comp", C.c_double), ("comp_kernel", C.c_int)]


DUMP_FIELDS = ["aq", "aq_scales", "bq", "bq_scales", "d_f", "raq", "raq_scale", "rbq",
               "rbq_scale", "row_stat", "col_stat", "a_red", "b_red", "a_red_scale",
               "b_red_scale", "a_keep", "b_keep"]


class XgDump(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in DUMP_FIELDS]


_V = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_D = C.c_double
_F = C.c_float

_SIGS = {
    "xg_last_error": (C.c_char_p, []),
    "xg_version": (_I, []),
    "xg_config_default": (XgConfig, []),
    "xg_device_ok": (_I, []),
    "xg_workspace_release": (_I, []),
    "xg_launch_count": (_I64, [_I]),
    "xg_gemm_max_inner": (_I, [_I]),
    "xg_quantize": (_I, [_V, _I, _I, _I, _I, _I, _V, _V, _V]),
    "xg_quantize_with_scales": (_I, [_V, _I, _I, _I, _I, _V, _I, _V, _V]),
    "xg_dequantize": (_I, [_V, _I, _I, _I, _V, _V, _V]),
    "xg_residual": (_I, [_V, _V, _I, _I, _I, _V, _V, _V]),
    "xg_dequant_product": (_I, [_V, _I, _I, _I, _V, _I, _V, _V, _V]),
    "xg_gemm_i8": (_I, [_V, _V, _I, _I, _I, _I, _I, _V, _V]),
    "xg_gemm_f32": (_I, [_V, _V, _I, _I, _I, _V, _V]),
    "xg_axpby": (_I, [_V, _F, _V, _F, _I64, _V]),
    "xg_subtract": (_I, [_V, _V, _V, _I64, _V]),
    "xg_add_inplace": (_I, [_V, _V, _I64, _V]),
    "xg_max_abs": (_I, [_V, _I64, _V, _V, _V]),
    "xg_reduce_count": (_I, [_V, _I, _I, _V, _D, _I, _D, _I, _V, _V, _V]),
    "xg_reduce_fill": (_I, [_V, _I, _I, _V, _D, _I, _D, _I, _V, _V, _V, _V]),
    "xg_quantize_csr": (_I, [_I, _I, _V, _V, _V, _I64, _I, _I, _I, _V, _V, _V]),
    "xg_csr_transpose_i8": (_I, [_I, _I, _V, _V, _V, _I64, _V, _V, _V, _V]),
    "xg_csr_transpose_f32": (_I, [_I, _I, _V, _V, _V, _I64, _V, _V, _V, _V]),
    "xg_spmm_i8": (_I, [_I, _I, _V, _V, _V, _V, _I, _I, _V, _V]),
    "xg_spmm_f32": (_I, [_I, _I, _V, _V, _V, _V, _I, _V, _V]),
    "xg_comp_model_set": (_I, [_D, _D, _D, _I]),
    "xg_comp_model_get": (None, [_V, _V, _V, _V]),
    "xg_calibrate_eta": (_I, [_I, _I, C.c_uint64, _I, _V, _V, _V, _V]),
    "xg_csr_from_dense_count": (_I, [_V, _I, _I, _V, _V, _V]),
    "xg_csr_from_dense_fill": (_I, [_V, _I, _I, _V, _V, _V, _V]),
    "xg_densify": (_I, [_I, _I, _V, _V, _V, _V, _V]),
    "xg_avg_vectors": (_I, [_V, _I, _I, _V, _V, _V]),
    "xg_abs_min_vectors": (_I, [_V, _I, _I, _V, _V, _V]),
    "xg_xigemm": (_I, [_V, _V, _V, _F, _F, _I, _I, _I, _V, _I, _V, _V, _V, _V]),
    "xg_shard_create": (_I, [_V, _V, _V, _F, _F, _I, _I, _V, _I, _I, _V, _I, _V, _V]),
    "xg_shard_step": (_I, [_V, _I, _V]),
    "xg_shard_exchange": (_I, [_V, _I, _I, _V, _V, _V, _V, _V]),
    "xg_shard_finish": (_I, [_V, _V, _V]),
    "xg_shard_destroy": (None, [_V]),
    "xg_shard_remote_cap": (_I, [_V]),
    "xg_shard_remote_needed": (_I, [_V]),
    "xg_shard_set_remote_cap": (_I, [_V, _I]),
    "xg_gemm_direct": (_I, [_V, _V, _I, _I, _I, _V, _V, _V]),
    "xg_gemm_direct_q": (_I, [_V, _I, _V, _V, _I, _V, _I, _I, _I, _I, _I, _V, _V]),
    "xg_xigemm_host": (_I, [_V, _V, _V, _F, _F, _I, _I, _I, _V, _I, _V, _V]),
    "xg_gemm_direct_host": (_I, [_V, _V, _I, _I, _I, _V, _V]),
    "xg_generate": (_I, [_I, _D, _D, C.c_uint64, _I64, _V, _V]),
}

_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    """Loads the in-tree shared object (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise XgError(f"{LIB_PATH} missing: run paper_2403_06924_b200.build.build() "
                              "(or __graft_entry__.build()) first")
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                f = getattr(handle, name)
                f.restype = res
                f.argtypes = args
            _lib = handle
        return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().xg_last_error().decode(errors="replace")
    if rc == 1:
        raise InvalidArgument(msg)
    if rc == 5:
        raise ShardRetry(msg)
    raise XgError(f"xigemm status {rc}: {msg}")


def exported_symbols() -> list[str]:
    return sorted(_SIGS)
