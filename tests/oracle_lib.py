"""TEST INFRASTRUCTURE: numpy/ctypes wrappers over the CPU oracle.

`Oracle(lib)` wraps either the C restatement (oracle/liboracle.so, symbols
xo_*) or the reference compiled from its own sources (oracle/_ref/
libxigemm_ref.so, symbols xr_*).  Both expose the same calling convention
(see oracle/xigemm_oracle.h); only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline/reference leg use this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libxigemm_ref.so")

F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
F64P = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
I8P = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
U8P = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class XoConfig(C.Structure):
    _fields_ = [("bits", C.c_int), ("threshold", C.c_double), ("density_limit", C.c_double),
                ("scheme", C.c_int), ("policy", C.c_int), ("rounding", C.c_int)]


class XoReport(C.Structure):
    _fields_ = [("density_a", C.c_double), ("density_b", C.c_double), ("path", C.c_int),
                ("nnz_a", C.c_int64), ("nnz_b", C.c_int64)]


_DUMP_FIELDS = [("aq", C.c_void_p), ("aq_scales", C.c_void_p), ("bq", C.c_void_p),
                ("bq_scales", C.c_void_p), ("d_int", C.c_void_p), ("d_f", C.c_void_p),
                ("raq", C.c_void_p), ("raq_scale", C.c_void_p), ("rbq", C.c_void_p),
                ("rbq_scale", C.c_void_p), ("row_stat", C.c_void_p), ("col_stat", C.c_void_p),
                ("a_mask", C.c_void_p), ("b_mask", C.c_void_p), ("a_red", C.c_void_p),
                ("a_red_scales", C.c_void_p), ("b_red", C.c_void_p),
                ("b_red_scales", C.c_void_p), ("dr1", C.c_void_p), ("dr2", C.c_void_p)]


class XoDump(C.Structure):
    _fields_ = _DUMP_FIELDS


def build_oracle(with_ref: bool = True) -> None:
    """Builds liboracle.so (always) and _ref (when the reference is present)."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    if with_ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)


def cfg(bits=8, threshold=0.5, density_limit=0.3, scheme=0, policy=1, rounding=1) -> XoConfig:
    """Defaults follow XigemmConfig (pipeline.hpp:19-28): Int8, M 0.5, s 0.3,
    PerTensor, MinRule, Nearest."""
    return XoConfig(bits, threshold, density_limit, scheme, policy, rounding)


class Oracle:
    def __init__(self, path: str, prefix: str):
        self.lib = C.CDLL(path)
        self.p = prefix
        self.is_ref = prefix == "xr"

    def _f(self, name):
        return getattr(self.lib, f"{self.p}_{name}")

    # --- pipeline -----------------------------------------------------------
    def xigemm(self, a, b, c=None, alpha=1.0, beta=0.0, config=None, reduce=True):
        config = config or cfg()
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        m, k = a.shape
        n = b.shape[1]
        out = np.zeros((m, n), np.float32)
        rep = XoReport()
        cp = None if c is None else np.ascontiguousarray(c, np.float32).ctypes.data
        f = self._f("xigemm")
        f.restype = C.c_int
        rc = f(C.c_void_p(a.ctypes.data), C.c_void_p(b.ctypes.data), C.c_void_p(cp),
               C.c_float(alpha), C.c_float(beta), m, k, n, C.byref(config), int(reduce),
               C.c_void_p(out.ctypes.data), C.byref(rep), *([None] if not self.is_ref else []))
        return rc, out, rep

    def gemm_direct(self, a, b, config=None):
        config = config or cfg()
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.zeros((a.shape[0], b.shape[1]), np.float32)
        rc = self._f("gemm_direct")(C.c_void_p(a.ctypes.data), C.c_void_p(b.ctypes.data),
                                    a.shape[0], a.shape[1], b.shape[1], C.byref(config),
                                    C.c_void_p(out.ctypes.data))
        return rc, out

    def dump(self, a, b, config):
        """All pipeline intermediates (oracle: xo_xigemm dump; ref: stage replay)."""
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        m, k = a.shape
        n = b.shape[1]
        vw = config.scheme == 1
        bufs = dict(
            aq=np.zeros((m, k), np.int8), aq_scales=np.zeros(m if vw else 1),
            bq=np.zeros((k, n), np.int8), bq_scales=np.zeros(n if vw else 1),
            d_int=np.zeros((m, n), np.int32), d_f=np.zeros((m, n), np.float32),
            raq=np.zeros((m, k), np.int8), raq_scale=np.zeros(1),
            rbq=np.zeros((k, n), np.int8), rbq_scale=np.zeros(1),
            row_stat=np.zeros(m, np.float32), col_stat=np.zeros(n, np.float32),
            a_mask=np.zeros((m, k), np.uint8), b_mask=np.zeros((k, n), np.uint8),
            a_red=np.zeros((m, k), np.int8), a_red_scales=np.zeros(m if vw else 1),
            b_red=np.zeros((k, n), np.int8), b_red_scales=np.zeros(n if vw else 1),
            dr1=np.zeros((m, n), np.int32), dr2=np.zeros((m, n), np.int32))
        d = XoDump(*[C.c_void_p(bufs[name].ctypes.data) for name, _ in _DUMP_FIELDS])
        if self.is_ref:
            rc = self.lib.xr_pipeline_dump(C.c_void_p(a.ctypes.data), C.c_void_p(b.ctypes.data),
                                           m, k, n, C.byref(config), C.byref(d))
        else:
            out = np.zeros((m, n), np.float32)
            rc = self.lib.xo_xigemm(C.c_void_p(a.ctypes.data), C.c_void_p(b.ctypes.data), None,
                                    C.c_float(1.0), C.c_float(0.0), m, k, n, C.byref(config), 1,
                                    C.c_void_p(out.ctypes.data), None, C.byref(d))
            bufs["result"] = out
        return rc, bufs

    # --- stages -------------------------------------------------------------
    def quantize(self, a, bits=8, scheme=0, rounding=1):
        a = np.ascontiguousarray(a, np.float32)
        r, c = a.shape
        q = np.zeros((r, c), np.int8)
        s = np.zeros(r if scheme == 1 else c if scheme == 2 else 1)
        rc = self._f("quantize")(C.c_void_p(a.ctypes.data), r, c, bits, scheme, rounding,
                                 C.c_void_p(q.ctypes.data), C.c_void_p(s.ctypes.data))
        return rc, q, s

    def quantize_with_scales(self, a, scales, bits=8, scheme=0, rounding=1):
        a = np.ascontiguousarray(a, np.float32)
        s = np.ascontiguousarray(scales, np.float64)
        r, c = a.shape
        q = np.zeros((r, c), np.int8)
        rc = self._f("quantize_with_scales")(C.c_void_p(a.ctypes.data), r, c, bits, scheme,
                                             C.c_void_p(s.ctypes.data), rounding,
                                             C.c_void_p(q.ctypes.data))
        return rc, q

    def dequantize(self, q, scales, scheme=0):
        q = np.ascontiguousarray(q, np.int8)
        s = np.ascontiguousarray(scales, np.float64)
        out = np.zeros(q.shape, np.float32)
        rc = self._f("dequantize")(C.c_void_p(q.ctypes.data), q.shape[0], q.shape[1], scheme,
                                   C.c_void_p(s.ctypes.data), C.c_void_p(out.ctypes.data))
        return rc, out

    def residual(self, a, q, scales, scheme=0):
        a = np.ascontiguousarray(a, np.float32)
        q = np.ascontiguousarray(q, np.int8)
        s = np.ascontiguousarray(scales, np.float64)
        out = np.zeros(a.shape, np.float32)
        rc = self._f("residual")(C.c_void_p(a.ctypes.data), C.c_void_p(q.ctypes.data), a.shape[0],
                                 a.shape[1], scheme, C.c_void_p(s.ctypes.data),
                                 C.c_void_p(out.ctypes.data))
        return rc, out

    def dequant_product(self, p, sa, sb, scheme_a=0, scheme_b=0):
        p = np.ascontiguousarray(p, np.int32)
        sa = np.ascontiguousarray(sa, np.float64)
        sb = np.ascontiguousarray(sb, np.float64)
        out = np.zeros(p.shape, np.float32)
        rc = self._f("dequant_product")(C.c_void_p(p.ctypes.data), p.shape[0], p.shape[1],
                                        scheme_a, C.c_void_p(sa.ctypes.data), scheme_b,
                                        C.c_void_p(sb.ctypes.data), C.c_void_p(out.ctypes.data))
        return rc, out

    def gemm_int(self, a, b, bits_a=8, bits_b=8):
        a = np.ascontiguousarray(a, np.int8)
        b = np.ascontiguousarray(b, np.int8)
        c = np.zeros((a.shape[0], b.shape[1]), np.int32)
        rc = self._f("gemm_int")(C.c_void_p(a.ctypes.data), C.c_void_p(b.ctypes.data), a.shape[0],
                                 a.shape[1], b.shape[1], bits_a, bits_b, C.c_void_p(c.ctypes.data))
        return rc, c

    def gemm_f32(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        c = np.zeros((a.shape[0], b.shape[1]), np.float32)
        rc = self._f("gemm_f32")(C.c_void_p(a.ctypes.data), C.c_void_p(b.ctypes.data), a.shape[0],
                                 a.shape[1], b.shape[1], C.c_void_p(c.ctypes.data))
        return rc, c

    def axpby(self, d, alpha, c, beta):
        d = np.array(d, np.float32, copy=True, order="C")
        c = np.ascontiguousarray(c, np.float32)
        if self.is_ref:
            rc = self.lib.xr_axpby(C.c_void_p(d.ctypes.data), C.c_float(alpha),
                                   C.c_void_p(c.ctypes.data), C.c_float(beta), d.shape[0],
                                   d.shape[1])
        else:
            rc = self.lib.xo_axpby(C.c_void_p(d.ctypes.data), C.c_float(alpha),
                                   C.c_void_p(c.ctypes.data), C.c_float(beta), C.c_int64(d.size))
        return rc, d

    def avg_vectors(self, d):
        return self._vec("avg_vectors", d)

    def abs_min_vectors(self, d):
        return self._vec("abs_min_vectors", d)

    def _vec(self, name, d):
        d = np.ascontiguousarray(d, np.float32)
        r = np.zeros(d.shape[0], np.float32)
        c = np.zeros(d.shape[1], np.float32)
        rc = self._f(name)(C.c_void_p(d.ctypes.data), d.shape[0], d.shape[1],
                           C.c_void_p(r.ctypes.data), C.c_void_p(c.ctypes.data))
        return rc, r, c

    def reduce(self, m, stat, thr, policy, scale_other=1.0, per_row=True):
        m = np.ascontiguousarray(m, np.float32)
        stat = np.ascontiguousarray(stat, np.float32)
        rows, cols = m.shape
        rp = np.zeros(rows + 1, np.int32)
        ci = np.zeros(max(1, rows * cols), np.int32)
        v = np.zeros(max(1, rows * cols), np.float32)
        nnz = C.c_int64(0)
        if self.is_ref:
            rc = self.lib.xr_reduce(C.c_void_p(m.ctypes.data), rows, cols,
                                    C.c_void_p(stat.ctypes.data), len(stat), C.c_double(thr),
                                    policy, C.c_double(scale_other), int(per_row),
                                    C.c_void_p(rp.ctypes.data), C.c_void_p(ci.ctypes.data),
                                    C.c_void_p(v.ctypes.data), C.byref(nnz))
        else:
            if len(stat) != (rows if per_row else cols):
                return 1, None, None, None
            rc = self.lib.xo_reduce(C.c_void_p(m.ctypes.data), rows, cols,
                                    C.c_void_p(stat.ctypes.data), C.c_double(thr), policy,
                                    C.c_double(scale_other), int(per_row),
                                    C.c_void_p(rp.ctypes.data), C.c_void_p(ci.ctypes.data),
                                    C.c_void_p(v.ctypes.data), C.byref(nnz))
        if rc:
            return rc, None, None, None
        return rc, rp, ci[: nnz.value].copy(), v[: nnz.value].copy()

    def quantize_csr(self, rows, cols, rp, ci, v, bits=8, scheme=0, rounding=1):
        rp = np.ascontiguousarray(rp, np.int32)
        ci = np.ascontiguousarray(ci if len(ci) else np.zeros(1, np.int32), np.int32)
        v = np.ascontiguousarray(v if len(v) else np.zeros(1, np.float32), np.float32)
        qv = np.zeros(max(1, int(rp[-1])), np.int8)
        s = np.zeros(rows if scheme == 1 else cols if scheme == 2 else 1)
        rc = self._f("quantize_csr")(rows, cols, C.c_void_p(rp.ctypes.data),
                                     C.c_void_p(ci.ctypes.data), C.c_void_p(v.ctypes.data), bits,
                                     scheme, rounding, C.c_void_p(qv.ctypes.data),
                                     C.c_void_p(s.ctypes.data))
        return rc, qv[: int(rp[-1])].copy(), s

    def spmm_int(self, rows, cols, rp, ci, v, d, d_bits=8):
        rp = np.ascontiguousarray(rp, np.int32)
        ci = np.ascontiguousarray(ci if len(ci) else np.zeros(1, np.int32), np.int32)
        v = np.ascontiguousarray(v if len(v) else np.zeros(1, np.int8), np.int8)
        d = np.ascontiguousarray(d, np.int8)
        out = np.zeros((rows, d.shape[1]), np.int32)
        rc = self._f("spmm_int")(rows, cols, C.c_void_p(rp.ctypes.data),
                                 C.c_void_p(ci.ctypes.data), C.c_void_p(v.ctypes.data),
                                 C.c_void_p(d.ctypes.data), d.shape[1], d_bits,
                                 C.c_void_p(out.ctypes.data))
        return rc, out

    def spmm_f32(self, rows, cols, rp, ci, v, d):
        rp = np.ascontiguousarray(rp, np.int32)
        ci = np.ascontiguousarray(ci if len(ci) else np.zeros(1, np.int32), np.int32)
        v = np.ascontiguousarray(v if len(v) else np.zeros(1, np.float32), np.float32)
        d = np.ascontiguousarray(d, np.float32)
        out = np.zeros((rows, d.shape[1]), np.float32)
        rc = self._f("spmm_f32")(rows, cols, C.c_void_p(rp.ctypes.data),
                                 C.c_void_p(ci.ctypes.data), C.c_void_p(v.ctypes.data),
                                 C.c_void_p(d.ctypes.data), d.shape[1],
                                 C.c_void_p(out.ctypes.data))
        return rc, out

    def csr_transpose_i8(self, rows, cols, rp, ci, v):
        rp = np.ascontiguousarray(rp, np.int32)
        nnz = int(rp[-1])
        ci = np.ascontiguousarray(ci if nnz else np.zeros(1, np.int32), np.int32)
        v = np.ascontiguousarray(v if nnz else np.zeros(1, np.int8), np.int8)
        trp = np.zeros(cols + 1, np.int32)
        tci = np.zeros(max(1, nnz), np.int32)
        tv = np.zeros(max(1, nnz), np.int8)
        rc = self._f("csr_transpose_i8")(rows, cols, C.c_void_p(rp.ctypes.data),
                                         C.c_void_p(ci.ctypes.data), C.c_void_p(v.ctypes.data),
                                         C.c_void_p(trp.ctypes.data), C.c_void_p(tci.ctypes.data),
                                         C.c_void_p(tv.ctypes.data))
        return rc, trp, tci[:nnz].copy(), tv[:nnz].copy()

    def generate(self, kind, p1, p2, seed, rows, cols):
        out = np.zeros((rows, cols), np.float32)
        f = self._f("generate")
        rc = f(kind, C.c_double(p1), C.c_double(p2), C.c_uint64(seed), rows, cols,
               C.c_void_p(out.ctypes.data))
        return rc, out


def random_dense(rows, cols, seed, lo=-1.0, hi=1.0):
    """tests/test_support.hpp:16-24 (via the C restatement)."""
    lib = C.CDLL(ORACLE_SO)
    out = np.zeros((rows, cols), np.float32)
    lib.xo_random_dense(rows, cols, C.c_uint64(seed), C.c_float(lo), C.c_float(hi),
                        C.c_void_p(out.ctypes.data))
    return out


def oracle() -> Oracle:
    if not os.path.exists(ORACLE_SO):
        build_oracle(with_ref=False)
    return Oracle(ORACLE_SO, "xo")


def reference() -> Oracle | None:
    if not os.path.exists(REF_SO):
        return None
    return Oracle(REF_SO, "xr")


def keep_mask(words, rows: int, k: int) -> np.ndarray:
    """Unpacks an xg_dump keep bitmask (rows x ceil(k/32) uint32 words, bit k % 32
    of word k / 32) into a rows x k bool array."""
    w = np.ascontiguousarray(np.asarray(words.cpu() if hasattr(words, "cpu") else words)).view(np.uint32)
    w = w.reshape(rows, -1)
    bits = np.unpackbits(w.view(np.uint8).reshape(rows, -1), axis=1, bitorder="little")
    return bits[:, :k].astype(bool)

